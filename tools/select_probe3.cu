// select_probe3.cu -- cycle cost of the bf16 selection phases as the stack
// kernel runs them (one CTA, warm): histogram clear, x load + 15-bit
// histogram, exact cut (tie and no-tie k), and the two row-list compactions
// (compact2 with per-index predicates vs compact2_16, 8 channels per lane).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2504_19449_b200/csrc -o tools/select_probe3 tools/select_probe3.cu
#include <cuda_bf16.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

__device__ long long g_stamp[16];
#define RSP_SEL_STAMP(i)                                  \
  do {                                                    \
    if (threadIdx.x == 0) {                               \
      long long c_;                                       \
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_)); \
      g_stamp[i] = c_;                                    \
    }                                                     \
  } while (0)
#include "rsp_select.cuh"

using namespace rsp;

__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

__global__ void __launch_bounds__(kThreads, 1) probe(const void* x, int n, int k, int a1, int b1, int reps,
                                                     long long* out, int* res, uint32_t zero) {
  extern __shared__ __align__(16) uint8_t sm[];
  const uint32_t sb = smem_base_pinned(sm);
  SelArea S;
  S.h1 = sb;
  S.cand = S.h1 + 4u * kBins;
  S.h2a = S.cand + 4u * kCandWords;
  S.h2b = S.h2a + 4u * 256;
  S.misc = S.h2b + 4u * 256;
  S.h16 = S.misc + 4u * kMiscWords;
  S.xs = S.h16 + 4u * kH16Words;
  S.zero = zero;
  const uint32_t lw = S.xs + ((2u * n + 15u) & ~15u);
  const uint32_t lu = lw + 8u * (a1 + 32);
  long long t[8];
  Cut cut;
  int nW = 0, nU = 0, nW2 = 0, nU2 = 0;
  for (int r = 0; r < reps; ++r) {
    sel_clear16(S);
    __syncthreads();
    t[0] = clk();
    sel_load16(x, n, S);
    t[1] = clk();
    if (threadIdx.x == 0) g_stamp[0] = t[1];
    cut = sel_cut16(n, k, S);
    t[2] = clk();
    compact2(
        S, 0, a1, 0, b1, [&](int j) { return in_cut(sel_key<true>(S, j), j, cut); },
        [&](int j) { return !in_cut(sel_key<true>(S, j), j, cut); },
        [&](int i, int j) { sts2(lw + 8u * i, static_cast<uint32_t>(j), sel_bits<true>(S, j)); },
        [&](int i, int j) { sts2(lu + 8u * i, static_cast<uint32_t>(j), sel_bits<true>(S, j)); }, &nW, &nU);
    t[3] = clk();
    compact2_16(
        S, cut, 0, a1, 0, b1,
        [&](bool p, int i, int j, uint32_t bits) { sts2_pred(p, lw + 8u * i, static_cast<uint32_t>(j), bits); },
        [&](bool p, int i, int j, uint32_t bits) { sts2_pred(p, lu + 8u * i, static_cast<uint32_t>(j), bits); }, &nW2, &nU2);
    t[4] = clk();
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) out[i] = t[i + 1] - t[i];
    res[0] = static_cast<int>(cut.T >> 16);
    res[1] = cut.jlim;
    res[2] = nW;
    res[3] = nU;
    res[4] = nW2;
    res[5] = nU2;
    res[6] = static_cast<int>(S.m(M_CNT));
    for (int i = 1; i < 9; ++i) out[8 + i] = g_stamp[i] ? g_stamp[i] - g_stamp[0] : -1;
  }
}

int main() {
  struct Case {
    int n, a1, b1;
  };
  const Case cases[] = {{4096, 341, 85}, {4096, 1365, 28}, {11008, 1224, 76}};
  for (const Case& c : cases) {
    const int n = c.n;
    std::vector<__nv_bfloat16> xb(n);
    srand(7);
    for (int i = 0; i < n; ++i) {
      const double u = (rand() + 0.5) / (RAND_MAX + 1.0) - 0.5;
      const double lap = (u < 0 ? 1 : -1) * log(1 - 2 * fabs(u));
      const double g = sqrt(-2 * log((rand() + 0.5) / (RAND_MAX + 1.0))) * cos(6.2831853 * rand() / RAND_MAX);
      xb[i] = __float2bfloat16(static_cast<float>(lap * exp(g)));
    }
    void* dxb;
    cudaMalloc(&dxb, n * 2);
    cudaMemcpy(dxb, xb.data(), n * 2, cudaMemcpyHostToDevice);
    long long* dout;
    int* dres;
    cudaMalloc(&dout, 64 * 8);
    cudaMemset(dout, 0, 64 * 8);
    cudaMalloc(&dres, 64 * 4);
    const size_t smem = 4u * (kBins + kCandWords + 512 + kMiscWords + kH16Words) + 2u * n + 16 + 8u * (n + 64);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (double s : {0.16, 0.202, 0.21, 0.25, 0.3}) {
      const int k = static_cast<int>(ceil(s * n));
      probe<<<1, kThreads, smem>>>(dxb, n, k, c.a1, c.b1, 4, dout, dres, 0u);
      long long o[24];
      int r[8];
      cudaMemcpy(o, dout, sizeof(o), cudaMemcpyDeviceToHost);
      cudaMemcpy(r, dres, sizeof(r), cudaMemcpyDeviceToHost);
      printf("n=%5d k=%5d A=%4d B=%3d | load+hist %5lld  cut %5lld  compact2 %5lld  compact2_16 %5lld cyc | key %d jlim %d cnt %d lists %d/%d vs %d/%d\n",
             n, k, c.a1, c.b1, o[0], o[1], o[2], o[3], r[0], r[1], r[6], r[2], r[3], r[4], r[5]);
      printf("      cut stamps: scan %lld  sync1 %lld  search %lld  sync2 %lld  tie-start %lld  tie-pass %lld  tie-sync %lld  end %lld\n", o[9], o[10], o[11], o[12], o[16], o[14], o[15], o[13]);
    }
    cudaFree(dxb);
    cudaFree(dout);
    cudaFree(dres);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
