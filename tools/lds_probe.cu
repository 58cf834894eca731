// lds_probe.cu -- cycles of the gather-count loop body in isolation (one CTA,
// 512 threads, keys in shared memory), to separate LDS / VOTE / sync costs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2504_19449_b200/csrc -o tools/lds_probe tools/lds_probe.cu
#include <stdio.h>

#include "rsp_select.cuh"

using namespace rsp;

__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int n, uint32_t bin, long long* out, uint32_t* sink) {
  __shared__ __align__(16) uint16_t xs[16384];
  for (int i = threadIdx.x; i < n; i += 512) xs[i] = static_cast<uint16_t>((i * 2654435761u) >> 16);
  __syncthreads();
  SelArea S;
  S.xs = smem_base_pinned(xs);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = n * warp / 16, r1 = n * (warp + 1) / 16;
  long long t[4];
  uint32_t mine = 0;
  for (int rep = 0; rep < 4; ++rep) {
    __syncthreads();
    t[rep] = clk();
    for (int j0 = r0; j0 < r1; j0 += 128) {
      uint32_t kq[4];
      if (MODE == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) kq[q] = j0 + 32 * q + lane < r1 ? sel_key<true>(S, j0 + 32 * q + lane) : 0u;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) kq[q] = j0 + 32 * q + lane < r1 ? (uint32_t(xs[j0 + 32 * q + lane]) << 16) & 0x7fffffffu : 0u;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        mine += __popc(__ballot_sync(0xffffffffu, j0 + 32 * q + lane < r1 && (kq[q] >> 19) == bin));
    }
  }
  __syncthreads();
  const long long te = clk();
  if (threadIdx.x == 0) {
    out[0] = t[1] - t[0];
    out[1] = t[2] - t[1];
    out[2] = t[3] - t[2];
    out[3] = te - t[3];
  }
  sink[threadIdx.x] = mine;
}

int main() {
  long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 64);
  cudaMalloc(&sink, 4096);
  long long h[4];
  for (int n : {4096, 11008}) {
    k<0><<<1, 512>>>(n, 0x7f0, d, sink);
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("n=%d asm-lds   : %lld %lld %lld %lld cycles per pass\n", n, h[0], h[1], h[2], h[3]);
    k<1><<<1, 512>>>(n, 0x7f0, d, sink);
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    printf("n=%d plain-lds : %lld %lld %lld %lld cycles per pass\n", n, h[0], h[1], h[2], h[3]);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
