// calib2.cu -- why does a tiny single-warp section between two barriers cost
// ~2k cycles inside sel_cut?  Variants: inline vs noinline, stamp via global
// store vs register.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2504_19449_b200/csrc -o tools/calib2 tools/calib2.cu
#include <stdio.h>

#include "rsp_device.cuh"

using namespace rsp;

__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

template <bool INL>
struct Sec;

__device__ __forceinline__ uint32_t section_body(uint32_t h, uint32_t need) {
  const int lane = threadIdx.x & 31;
  uint32_t r = 0;
  if ((threadIdx.x >> 5) == 0) {
    const uint32_t c = lane < 8 ? lds(h + 4u * (7 - lane)) : 0u;
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t hit = __ballot_sync(0xffffffffu, lane < 8 && inc - c < need && need <= inc);
    const int src = __ffs(hit) - 1;
    r = __shfl_sync(0xffffffffu, inc - c, src);
    if (lane == 0) sts(h + 64u, r);
  }
  __syncthreads();
  return lds(h + 64u) + r;
}

__device__ __noinline__ uint32_t section_noinline(uint32_t h, uint32_t need) { return section_body(h, need); }

template <int MODE>
__global__ void __launch_bounds__(512, 1) kern(long long* out, uint32_t* sink, uint32_t need) {
  __shared__ uint32_t h[64];
  if (threadIdx.x < 64) h[threadIdx.x] = threadIdx.x;
  __syncthreads();
  const uint32_t hb = smem_base_pinned(h);
  uint32_t acc = 0;
  long long t[5];
  for (int r = 0; r < 5; ++r) {
    __syncthreads();
    t[r] = clk();
    if (MODE == 0) acc += section_body(hb, need + r);
    else acc += section_noinline(hb, need + r);
  }
  __syncthreads();
  const long long te = clk();
  if (threadIdx.x == 0) {
    for (int r = 0; r < 4; ++r) out[r] = t[r + 1] - t[r];
    out[4] = te - t[4];
  }
  sink[threadIdx.x] = acc;
}

int main() {
  long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 64);
  cudaMalloc(&sink, 4096);
  long long h[5];
  for (int rep = 0; rep < 2; ++rep) {
    kern<0><<<1, 512>>>(d, sink, 100);
    cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
    printf("inline  : %lld %lld %lld %lld %lld\n", h[0], h[1], h[2], h[3], h[4]);
    kern<1><<<1, 512>>>(d, sink, 100);
    cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
    printf("noinline: %lld %lld %lld %lld %lld\n", h[0], h[1], h[2], h[3], h[4]);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
