// prefetch_probe.cu -- does an L2 prefetch issued ahead make a later read an
// L2 hit on B200?  Region R (32 MB, fresh each rep) is
//   (0) read cold,
//   (1) prefetched by prefetch.global.L2::evict_last (one per 128-B line), then read,
//   (2) prefetched by cp.async.bulk.prefetch.L2 (one per 4 KB), then read,
//   (3) read once (warm), then read again.
// The reads are timed on their own (events around the read kernel only).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/prefetch_probe tools/prefetch_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                             \
  do {                                                                    \
    cudaError_t e = (x);                                                  \
    if (e != cudaSuccess) {                                               \
      printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                            \
    }                                                                     \
  } while (0)

__device__ __forceinline__ uint4 ldg_nc(const void* p) {
  uint4 u;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "l"(p));
  return u;
}

__device__ unsigned long long g_t0, g_t1;
__global__ void __launch_bounds__(512) read_kernel(const uint4* p, size_t nvec, float* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0) atomicMin(&g_t0, t);
  uint32_t acc = 0;
  const size_t tot = static_cast<size_t>(gridDim.x) * blockDim.x;
  size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 7 * tot < nvec; i += 8 * tot) {
    uint4 u[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) u[q] = ldg_nc(p + i + q * tot);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc ^= u[q].x ^ u[q].w;
  }
  if (acc == 0x12345678u) out[0] = 1.f;
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (threadIdx.x == 0) atomicMax(&g_t1, t);
}

__global__ void pf_line(const uint8_t* p, size_t bytes) {
  for (size_t o = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 128; o < bytes;
       o += static_cast<size_t>(gridDim.x) * blockDim.x * 128)
    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p + o));
}

__global__ void pf_bulk(const uint8_t* p, size_t bytes) {
  for (size_t o = (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4096; o < bytes;
       o += static_cast<size_t>(gridDim.x) * blockDim.x * 4096)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + o), "r"(4096u) : "memory");
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t BUF = size_t(4) << 30, R = size_t(32) << 20;
  uint8_t* W;
  CK(cudaMalloc(&W, BUF));
  CK(cudaMemset(W, 1, BUF));
  float* out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"cold", "prefetch.L2 lines", "bulk prefetch 4KB", "warm re-read"};
  for (int mode = 0; mode < 4; ++mode) {
    double tot = 0;
    const int reps = 20;
    for (int r = 0; r < reps; ++r) {
      const uint8_t* p = W + (static_cast<size_t>(r + mode * reps) * R) % (BUF - R);
      // evict: stream 256 MB of other data through L2
      const size_t ev = size_t(256) << 20;
      const size_t eoff = (static_cast<size_t>((r + 50) * 97 % 12) * ev) % (BUF - ev);
      read_kernel<<<sms, 512>>>(reinterpret_cast<const uint4*>(W + eoff), ev / 16, out);
      if (mode == 1) pf_line<<<sms, 512>>>(p, R);
      if (mode == 2) pf_bulk<<<sms, 128>>>(p, R);
      if (mode == 3) read_kernel<<<sms, 512>>>(reinterpret_cast<const uint4*>(p), R / 16, out);
      CK(cudaDeviceSynchronize());
      unsigned long long big = ~0ull, zero = 0;
      CK(cudaMemcpyToSymbol(g_t0, &big, 8));
      CK(cudaMemcpyToSymbol(g_t1, &zero, 8));
      read_kernel<<<sms, 512>>>(reinterpret_cast<const uint4*>(p), R / 16, out);
      CK(cudaDeviceSynchronize());
      unsigned long long a, b;
      CK(cudaMemcpyFromSymbol(&a, g_t0, 8));
      CK(cudaMemcpyFromSymbol(&b, g_t1, 8));
      tot += (b - a) * 1e-6;  // ns -> ms
    }
    const double us = tot * 1e3 / reps;
    printf("%-20s 32 MB read (in-kernel globaltimer span): %.2f us  (%.0f GB/s)\n", names[mode], us, R / us / 1e3);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
