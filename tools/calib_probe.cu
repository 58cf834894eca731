// calib_probe.cu -- ground-truth cycle costs on this B200 for one CTA of 512
// threads: dependent IADD, __syncthreads, dependent LDS, dependent SHFL,
// VOTE throughput.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/calib_probe tools/calib_probe.cu
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

__global__ void __launch_bounds__(512, 1) calib(int iters, long long* out, uint32_t* sink, uint32_t seed) {
  __shared__ uint32_t sm[4096];
  for (int i = threadIdx.x; i < 4096; i += 512) sm[i] = (i * 7 + seed) & 4095;
  __syncthreads();
  uint32_t v = threadIdx.x ^ seed;
  long long t0 = clk();
  for (int i = 0; i < iters; ++i) asm volatile("add.u32 %0, %0, %1;" : "+r"(v) : "r"(seed));
  long long t1 = clk();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t2 = clk();
  uint32_t p = threadIdx.x;
  for (int i = 0; i < iters; ++i) p = sm[p & 4095];
  long long t3 = clk();
  for (int i = 0; i < iters; ++i) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31);
  long long t4 = clk();
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) acc += __popc(__ballot_sync(0xffffffffu, ((v + i) & 1) != 0));
  long long t5 = clk();
  // independent LDS throughput: 8 loads per iteration
  uint32_t a2 = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) a2 += sm[(threadIdx.x * 8 + q + i) & 4095];
  }
  long long t6 = clk();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0);
    out[1] = (t2 - t1);
    out[2] = (t3 - t2);
    out[3] = (t4 - t3);
    out[4] = (t5 - t4);
    out[5] = (t6 - t5);
  }
  sink[threadIdx.x] = v + p + acc + a2;
}

int main() {
  long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 64);
  cudaMalloc(&sink, 4096);
  long long h[6];
  for (int r = 0; r < 3; ++r) {
    calib<<<1, 512>>>(100, d, sink, r);
    cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
    printf("per-iteration cycles: dep IADD %.1f | syncthreads %.1f | dep LDS %.1f | dep SHFL %.1f | ballot+popc %.1f | 8 indep LDS %.1f\n",
           h[0] / 100.0, h[1] / 100.0, h[2] / 100.0, h[3] / 100.0, h[4] / 100.0, h[5] / 100.0);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
