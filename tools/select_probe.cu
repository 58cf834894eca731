// select_probe.cu -- per-phase clock64 cost of the production selector
// (rsp_select.cuh) run by 148 CTAs at once, x resident in L2.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2504_19449_b200/csrc -o select_probe select_probe.cu
#include <cuda_bf16.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <functional>
#include <vector>
#include <math.h>
#include <string.h>

#define RSP_SEL_DEBUG(level, prefix, need, cnt, extra) \
  if (blockIdx.x == 0 && threadIdx.x == 0 && dbg) printf("  L%d prefix=%08x need=%u cnt=%u cc=%u\n", level, prefix, need, cnt, extra);
__device__ int dbg;
#include "rsp_select.cuh"

using namespace rsp;


__global__ void __launch_bounds__(512, 1) probe(const void* x, int bf16, int n, int k, long long* out, int* sink) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t sb = smem_base_pinned(smem);
  SelSmem ss;
  ss.hist = sb;
  ss.cand = sb + 4u * kHistBins;
  ss.misc = ss.cand + 4u * kCandWords;
  ss.keys = ss.misc + 4u * kMiscWords;
  long long t0 = clock64();
  sel_clear(ss);
  __syncthreads();
  long long t1 = clock64();
  sel_load(x, bf16 != 0, n, ss, true);
  long long t2 = clock64();

  long long t3 = clock64();
  SelResult r = sel_resolve(n, k, bf16 != 0, ss);
  long long t4 = clock64();
  int acc = 0;
  sel_count(n, r, ss);
  const uint32_t lo = (uint32_t)(k * 4 / 9), hi = (uint32_t)(k * 5 / 9);
  sel_range_emit(n, r, ss, true, lo, hi, [&](int j, uint32_t bits, uint32_t i) { acc += j + (int)i; });
  sel_range_emit(n, r, ss, false, 20, 40, [&](int j, uint32_t bits, uint32_t i) { acc += j + (int)i; });
  __syncthreads();
  long long t5 = clock64();
  if (acc == 123456789) sink[0] = acc;
  if (threadIdx.x == 0) {
    long long* o = out + blockIdx.x * 8;
    o[0] = t1 - t0; o[1] = t2 - t1; o[2] = t3 - t2; o[3] = t4 - t3; o[4] = t5 - t4; o[5] = r.T; o[6] = r.need;
  }
}

int main() {
  const int grid = 148;
  for (int n : {4096, 11008}) {
    for (int bf16 = 0; bf16 < 2; ++bf16) {
      std::vector<float> xf(n);
      srand(1);
      for (auto& v : xf) {  // Laplace(0,1) * LogNormal(0,1)
        const float u = (rand() + 0.5f) / (RAND_MAX + 1.0f) - 0.5f;
        const float lap = (u < 0 ? 1.f : -1.f) * logf(1.f - 2.f * fabsf(u));
        const float u1 = (rand() + 0.5f) / (RAND_MAX + 1.0f), u2 = (rand() + 0.5f) / (RAND_MAX + 1.0f);
        v = lap * expf(sqrtf(-2.f * logf(u1)) * cosf(6.2831853f * u2));
      }
      std::vector<uint16_t> xb(n);
      std::vector<uint32_t> keys(n);
      for (int i = 0; i < n; ++i) {
        uint32_t u; memcpy(&u, &xf[i], 4); xb[i] = u >> 16;
        keys[i] = (bf16 ? (u & 0xffff0000u) : u) & 0x7fffffffu;
      }
      std::vector<uint32_t> sk = keys;
      std::sort(sk.begin(), sk.end(), std::greater<uint32_t>());
      const uint32_t T_ref = sk[n / 4 - 1];
      int gt = 0; for (auto kk : keys) gt += kk > T_ref;
      const long long need_ref = n / 4 - gt;
      void* dx;
      cudaMalloc(&dx, n * 4);
      cudaMemcpy(dx, bf16 ? (void*)xb.data() : (void*)xf.data(), n * (bf16 ? 2 : 4), cudaMemcpyHostToDevice);
      long long* dout;
      int* sink;
      cudaMalloc(&dout, 8192 * 8);
      cudaMalloc(&sink, 4);
      const size_t smem = 4 * (kHistBins + kCandWords + kMiscWords) + 4 * n;
      cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      { int one = 1; cudaMemcpyToSymbol(dbg, &one, 4); probe<<<1, 512, smem>>>(dx, bf16, n, n / 4, dout, sink); cudaDeviceSynchronize(); one = 0; cudaMemcpyToSymbol(dbg, &one, 4); }
      for (int it = 0; it < 5; ++it) probe<<<grid, 512, smem>>>(dx, bf16, n, n / 4, dout, sink);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      for (int it = 0; it < 100; ++it) probe<<<grid, 512, smem>>>(dx, bf16, n, n / 4, dout, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      std::vector<long long> h(8192);
      cudaMemcpy(h.data(), dout, h.size() * 8, cudaMemcpyDeviceToHost);
      double m[5] = {0};
      for (int b = 0; b < grid; ++b) for (int q = 0; q < 5; ++q) m[q] += h[b * 8 + q] / (double)grid;
      printf("n=%5d bf16=%d kernel %.2f us | cycles clear %.0f load %.0f hist %.0f resolve %.0f count+ranges %.0f | T=%llx need=%lld\n",
             n, bf16, ms * 10.0, m[0], m[1], m[2], m[3], m[4], h[5], h[6]);
      printf("   reference T=%x need=%lld  (whole-bin cut T=prefix-1,need=0 is equivalent)\n", T_ref, need_ref);
      cudaFree(dx); cudaFree(dout); cudaFree(sink);
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
