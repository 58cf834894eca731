// icache_probe.cu -- is straight-line (run-once) code fetch-bound?  Compare
// N unrolled distinct instructions vs the same count in a small loop,
// executed by 1 warp and by 8 warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/icache_probe tools/icache_probe.cu
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

template <int N>
__device__ __forceinline__ uint32_t straight(uint32_t v, uint32_t s) {
#pragma unroll
  for (int i = 0; i < N; ++i) v = (v ^ (s + i * 0x9E3779B9u)) * 3u + i;  // distinct immediates: no folding
  return v;
}

template <int WARPS>
__global__ void k(long long* out, uint32_t* sink, uint32_t s, int iters) {
  uint32_t v = threadIdx.x;
  long long t0 = 0, t1 = 0, t2 = 0, t3 = 0;
  if ((threadIdx.x >> 5) < WARPS) {
    t0 = clk();
    v = straight<1024>(v, s);
    t1 = clk();
    v = straight<1024>(v, s + 1);  // second copy: also cold
    t2 = clk();
    for (int i = 0; i < iters; ++i) v = (v ^ (s + i * 0x9E3779B9u)) * 3u + i;
    t3 = clk();
  }
  if (threadIdx.x == 0) {
    out[0] = t1 - t0;
    out[1] = t2 - t1;
    out[2] = t3 - t2;
  }
  sink[threadIdx.x] = v;
}

int main() {
  long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 64);
  cudaMalloc(&sink, 4096);
  long long h[3];
  for (int rep = 0; rep < 2; ++rep) {
    k<1><<<1, 256>>>(d, sink, 7, 1024);
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("1 warp : straight 1024 ops %lld cyc, again %lld cyc, loop 1024 iters %lld cyc\n", h[0], h[1], h[2]);
    k<8><<<1, 256>>>(d, sink, 7, 1024);
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("8 warps: straight 1024 ops %lld cyc, again %lld cyc, loop 1024 iters %lld cyc\n", h[0], h[1], h[2]);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
