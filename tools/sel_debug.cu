// sel_debug.cu -- run the production selector on a dumped fp32 vector and print S.
#include <cstdio>
#include <vector>
#define RSP_SEL_DEBUG(level, prefix, need, cnt, extra) \
  if (threadIdx.x == 0) printf("  L%d prefix=%08x need=%u cnt=%u cc=%u\n", level, prefix, need, cnt, extra);
#include "rsp_select.cuh"
using namespace rsp;
__global__ void __launch_bounds__(512, 1) k(const float* x, int n, int kk, int* kept, unsigned* keys_out) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t sb = smem_base_pinned(smem);
  SelSmem ss;
  ss.hist = sb; ss.cand = sb + 4u * kHistBins; ss.misc = ss.cand + 4u * kCandWords; ss.keys = ss.misc + 4u * kMiscWords;
  sel_clear(ss);
  __syncthreads();
  sel_load(x, false, n, ss, true);
  for (int j = threadIdx.x; j < n; j += 512) keys_out[j] = lds(ss.keys + 4u * j);
  const SelResult sr = sel_resolve(n, kk, false, ss);
  if (threadIdx.x == 0) printf("T=%08x need=%u\n", sr.T, sr.need);
  sel_count(n, sr, ss);
  if (threadIdx.x == 0) for (int c = 110; c < 125; ++c) { unsigned pk = lds(ss.cand + 4u * c); printf("chunk %d gt_pre %u tie_pre %u\n", c, pk & 0xffff, pk >> 16); }
  sel_range_emit(n, sr, ss, true, 0u, (uint32_t)kk, [&](int j, uint32_t bits, uint32_t i) { kept[i] = j; });
}
int main() {
  const int n = 4096, kk = 31;
  std::vector<float> h(n);
  FILE* f = fopen("tools/x_sign_dups.bin", "rb"); fread(h.data(), 4, n, f); fclose(f);
  float* dx; int* dk; unsigned* dkeys;
  cudaMalloc(&dx, n * 4); cudaMalloc(&dk, 64 * 4); cudaMalloc(&dkeys, n * 4);
  cudaMemcpy(dx, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemset(dk, 0xff, 64 * 4);
  size_t smem = 4 * (kHistBins + kCandWords + kMiscWords) + 4 * n;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<1, 512, smem>>>(dx, n, kk, dk, dkeys);
  cudaDeviceSynchronize();
  std::vector<int> hk(64); std::vector<unsigned> keys(n);
  cudaMemcpy(hk.data(), dk, 64 * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(keys.data(), dkeys, n * 4, cudaMemcpyDeviceToHost);
  printf("S:"); for (int i = 0; i < kk; ++i) printf(" %d", hk[i]); printf("\n");
  printf("keys 3840 %08x 3841 %08x 3410 %08x 492 %08x\n", keys[3840] & 0x7fffffff, keys[3841] & 0x7fffffff, keys[3410] & 0x7fffffff, keys[492] & 0x7fffffff);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
