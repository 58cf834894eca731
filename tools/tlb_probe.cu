// tlb_probe.cu -- does touching fresh address ranges cost (TLB reach)?
// Graph of 64 launches, each a flat read of B bytes from a chunk that rotates
// over a span of S bytes (S from 256 MB to 16 GB).  Chunks are consecutive, so
// every launch reads data not in L2 once S > 2x L2; only TLB reach differs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tlb_probe tools/tlb_probe.cu
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

// gathered: each CTA reads `rows` rows of `seg` bytes at stride `stride` (like W rows of one column tile)
__global__ void __launch_bounds__(512, 1) read_kernel(const uint8_t* p, size_t bytes, size_t stride, float* out) {
  uint32_t acc = 0;
  const size_t nvec = bytes / 16;
  const size_t tot = static_cast<size_t>(gridDim.x) * blockDim.x;
  size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  // scatter the flat index over the span: vector i -> row (i / 64) * stride + (i % 64) * 16 (1 KB rows)
  for (; i + 7 * tot < nvec; i += 8 * tot) {
    uint4 u[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const size_t v = i + q * tot;
      u[q] = ldg_nc(p + (v >> 6) * stride + (v & 63) * 16);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) acc ^= u[q].x ^ u[q].w;
  }
  if (acc == 0x12345678u) out[0] = 1.f;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t MAXB = size_t(16) << 30;
  uint8_t* W;
  CK(cudaMalloc(&W, MAXB));
  CK(cudaMemset(W, 1, MAXB));
  float* out;
  CK(cudaMalloc(&out, 64));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t bytes = size_t(16) << 20;  // 16 MB per launch
  const int L = 64;
  for (size_t span_mb : {256, 1024, 4096, 16384}) {
    for (size_t stride : {size_t(1024), size_t(8192), size_t(65536)}) {
      // each launch: bytes/1KB rows at `stride`, so it spans bytes/1024*stride
      const size_t per = bytes / 1024 * stride;
      const size_t span = span_mb << 20;
      if (per > span) continue;
      const int chunks = static_cast<int>(span / per);
      cudaGraph_t g;
      cudaGraphExec_t ge;
      CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      for (int i = 0; i < L; ++i)
        read_kernel<<<sms, 512, 0, s>>>(W + static_cast<size_t>(i % chunks) * per, bytes, stride, out);
      CK(cudaStreamEndCapture(s, &g));
      CK(cudaGraphInstantiate(&ge, g, 0));
      for (int w = 0; w < 2; ++w) CK(cudaGraphLaunch(ge, s));
      CK(cudaStreamSynchronize(s));
      CK(cudaEventRecord(e0, s));
      for (int r = 0; r < 5; ++r) CK(cudaGraphLaunch(ge, s));
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1e3 / (5 * L);
      printf("span %6zu MB  row stride %6zu  chunks %4d : %.2f us per 16 MB launch  %.0f GB/s\n", span_mb, stride,
             chunks, us, bytes / us / 1e3);
      cudaGraphExecDestroy(ge);
      cudaGraphDestroy(g);
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
