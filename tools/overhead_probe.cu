// overhead_probe.cu -- fixed per-linear costs on B200 that bound a decode stack:
//   (a) back-to-back kernels in a CUDA graph (148 CTAs x 512 thr, 100 KB smem),
//       plain vs programmatic dependent launch (PDL), empty bodies;
//   (b) one persistent kernel crossing N grid barriers (148 CTAs);
//   (c) contiguous read of B bytes per launch in a graph of 64 launches
//       (fresh bytes every launch), with PDL: effective GB/s vs B.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/overhead_probe tools/overhead_probe.cu
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

__device__ __forceinline__ void gdc_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void gdc_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__global__ void __launch_bounds__(512, 1) empty_kernel(int pdl, float* out) {
  extern __shared__ float sm[];
  if (pdl) {
    gdc_wait();
    gdc_launch();
  }
  if (threadIdx.x == 0) sm[0] = blockIdx.x;
  __syncthreads();
  if (sm[0] == -1.f) out[0] = 1.f;
}

__device__ __forceinline__ uint4 ldg_nc(const void* p) {
  uint4 u;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "l"(p));
  return u;
}

__global__ void __launch_bounds__(512, 1) read_kernel(const uint4* p, size_t nvec, int pdl, float* out) {
  if (pdl) {
    gdc_wait();
    gdc_launch();
  }
  uint32_t acc = 0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < nvec; i += 8 * stride) {
    uint4 u[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) u[q] = ldg_nc(p + i + q * stride);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc ^= u[q].x ^ u[q].y ^ u[q].z ^ u[q].w;
  }
  for (; i < nvec; i += stride) {
    uint4 u = ldg_nc(p + i);
    acc ^= u.x ^ u.y ^ u.z ^ u.w;
  }
  if (acc == 0x12345678u) out[0] = 1.f;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(512, 1) barrier_kernel(unsigned* bar, int n, int spin_ns) {
  // bar[0] = arrivals (monotone), target = (i+1)*grid
  for (int i = 0; i < n; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(bar, 1u);
      const unsigned target = (i + 1) * gridDim.x;
      while (ld_acquire(bar) < target) {
        if (spin_ns) __nanosleep(spin_ns);
      }
    }
    __syncthreads();
  }
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float* out;
  CK(cudaMalloc(&out, 64));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int N = 224;
  CK(cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  auto launch = [&](auto kern, size_t smem, bool pdl, auto... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, kern, args...));
  };
  auto time_graph = [&](auto body) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    body();
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int w = 0; w < 3; ++w) CK(cudaGraphLaunch(ge, s));
    CK(cudaStreamSynchronize(s));
    const int reps = 10;
    CK(cudaEventRecord(e0, s));
    for (int r = 0; r < reps; ++r) CK(cudaGraphLaunch(ge, s));
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    return ms * 1e3 / reps;
  };
  for (int pdl = 0; pdl < 2; ++pdl) {
    const float us = time_graph([&] {
      for (int i = 0; i < N; ++i) launch(empty_kernel, 100 * 1024, pdl != 0, pdl, out);
    });
    printf("graph_empty pdl=%d  %.3f us/kernel\n", pdl, us / N);
  }
  unsigned* bar;
  CK(cudaMalloc(&bar, 64));
  for (int spin : {0, 32, 100}) {
    CK(cudaMemset(bar, 0, 64));
    barrier_kernel<<<sms, 512, 0, s>>>(bar, 10, spin);
    CK(cudaStreamSynchronize(s));
    CK(cudaMemset(bar, 0, 64));
    CK(cudaEventRecord(e0, s));
    barrier_kernel<<<sms, 512, 0, s>>>(bar, 1000, spin);
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("grid_barrier spin=%d  %.3f us/barrier\n", spin, ms * 1e3 / 1000);
  }
  const size_t BUF = size_t(4) << 30;
  uint8_t* W;
  CK(cudaMalloc(&W, BUF));
  CK(cudaMemset(W, 1, BUF));
  for (size_t mb : {1, 2, 4, 8, 16, 33, 64}) {
    const size_t bytes = mb << 20;
    const int L = 64;
    for (int pdl = 0; pdl < 2; ++pdl) {
      const float us = time_graph([&] {
        for (int i = 0; i < L; ++i) {
          const uint4* p = reinterpret_cast<const uint4*>(W + (size_t(i) * bytes) % (BUF - bytes));
          launch(read_kernel, 0, pdl != 0, p, bytes / 16, pdl, out);
        }
      });
      printf("graph_read %3zu MB pdl=%d  %.2f us/launch  %.0f GB/s\n", mb, pdl, us / L, bytes / (us / L) / 1e3);
    }
  }
  CK(cudaDeviceSynchronize());
  printf("status ok\n");
  return 0;
}
