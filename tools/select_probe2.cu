// select_probe2.cu -- cycle cost of the selection phases, cold vs warm
// (same kernel code run R times in one CTA), and of match.any vs a
// ballot-built peer mask.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2504_19449_b200/csrc -o tools/select_probe2 tools/select_probe2.cu
#include <cuda_bf16.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <cstring>
#include <vector>

__device__ long long g_stamp[16];
#define RSP_SEL_STAMP_OFF(i)                                              \
  do {                                                                \
    if (threadIdx.x == 0) {                                           \
      long long c_;                                                   \
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_));             \
      g_stamp[i] = c_;                                                \
    }                                                                 \
  } while (0)
#include "rsp_select.cuh"

using namespace rsp;

__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

template <bool XBF>
__global__ void __launch_bounds__(kThreads, 1) probe(const void* x, int n, int k, int reps, long long* out,
                                                     int* cut_out) {
  extern __shared__ __align__(16) uint8_t sm[];
  const uint32_t sb = smem_base_pinned(sm);
  SelArea S;
  S.h1 = sb;
  S.cand = S.h1 + 4u * kBins;
  S.h2a = S.cand + 4u * kCandWords;
  S.h2b = S.h2a + 4u * 256;
  S.misc = S.h2b + 4u * 256;
  S.xs = S.misc + 4u * kMiscWords;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    const long long t0 = clk();
    sel_clear(S);
    __syncthreads();
    const long long t1 = clk();
    sel_load<XBF>(x, n, S, true);
    const long long t2 = clk();
    const Cut c = sel_cut<XBF>(n, k, S);
    __syncthreads();
    const long long t3 = clk();
    if (threadIdx.x == 0) {
      out[r * 4 + 0] = t1 - t0;
      out[r * 4 + 1] = t2 - t1;
      out[r * 4 + 2] = t3 - t2;
      out[r * 4 + 3] = t3 - t0;
      for (int i = 0; i < 7; ++i) out[32 + i] = g_stamp[i] ? g_stamp[i] - t2 : -1;
      for (int i = 0; i < 7; ++i) g_stamp[i] = 0;
      cut_out[0] = static_cast<int>(c.T);
      cut_out[1] = c.jlim;
    }
  }
}

int main() {
  const int ns[] = {4096, 11008};
  for (int n : ns) {
    std::vector<float> x(n);
    srand(1);
    for (int i = 0; i < n; ++i) {
      const double u = (rand() + 0.5) / (RAND_MAX + 1.0) - 0.5;
      const double lap = (u < 0 ? 1 : -1) * log(1 - 2 * fabs(u));
      const double g = sqrt(-2 * log((rand() + 0.5) / (RAND_MAX + 1.0))) * cos(6.2831853 * rand() / RAND_MAX);
      x[i] = static_cast<float>(lap * exp(g));
    }
    std::vector<__nv_bfloat16> xb(n);
    for (int i = 0; i < n; ++i) xb[i] = __float2bfloat16(x[i]);
    void *dx, *dxb;
    cudaMalloc(&dx, n * 4);
    cudaMalloc(&dxb, n * 2);
    cudaMemcpy(dx, x.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dxb, xb.data(), n * 2, cudaMemcpyHostToDevice);
    long long* dout;
    int* dcut;
    cudaMalloc(&dout, 64 * 8);
    cudaMemset(dout, 0, 64 * 8);
    cudaMalloc(&dcut, 8);
    const size_t smem = 4u * (kBins + kCandWords + 512 + kMiscWords) + 4u * n + 16;
    cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int xbf = 1; xbf >= 0; --xbf) {
      const int reps = 4;
      if (xbf)
        probe<true><<<1, kThreads, smem>>>(dxb, n, n / 4, reps, dout, dcut);
      else
        probe<false><<<1, kThreads, smem>>>(dx, n, n / 4, reps, dout, dcut);
      long long h[64];
      cudaMemcpy(h, dout, reps * 4 * 8, cudaMemcpyDeviceToHost);
      printf("n=%d xbf=%d:", n, xbf);
      for (int r = 0; r < reps; ++r)
        printf("  [zero %lld load %lld cut %lld total %lld]", h[r * 4], h[r * 4 + 1], h[r * 4 + 2], h[r * 4 + 3]);
      int cut[2];
      cudaMemcpy(cut, dcut, 8, cudaMemcpyDeviceToHost);
      std::vector<uint32_t> key(n);
      for (int i = 0; i < n; ++i) {
        float f = xbf ? __bfloat162float(xb[i]) : x[i];
        uint32_t u;
        memcpy(&u, &f, 4);
        key[i] = u & 0x7fffffffu;
      }
      std::vector<int> idx(n);
      for (int i = 0; i < n; ++i) idx[i] = i;
      std::sort(idx.begin(), idx.end(), [&](int a, int b) { return key[a] != key[b] ? key[a] > key[b] : a < b; });
      const int kq = n / 4;
      int cntS = 0;
      for (int j = 0; j < n; ++j) cntS += key[j] > (uint32_t)cut[0] || (key[j] == (uint32_t)cut[0] && j < cut[1]);
      bool ok = cntS == kq;
      for (int q = 0; q < kq && ok; ++q) {
        const int j = idx[q];
        ok = key[j] > (uint32_t)cut[0] || (key[j] == (uint32_t)cut[0] && j < cut[1]);
      }
      printf("  cut_check=%s", ok ? "ok" : "MISMATCH");
      cudaMemcpy(h, dout, 64 * 8, cudaMemcpyDeviceToHost);
      printf("\n   cut stamps:");
      for (int i = 0; i < 7; ++i) printf(" %d:%lld", i, h[32 + i]);
      printf("\n");
    }
    cudaFree(dx);
    cudaFree(dxb);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
