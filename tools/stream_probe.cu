// stream_probe.cu -- how fast can 148 CTAs stream gathered weight rows?
// (a) cp.async.bulk 1-D copies of `seg` bytes into an smem ring (producer lane
//     per copy, `stages` x 16 KB), consumers FMA from smem;
// (b) LDG.128 from each lane, `unroll` rows in flight per warp.
// Rows are picked by a pseudo-random permutation (gathered, like S).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  }
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// rows: [nrows][row_elems] bf16; each CTA handles rows_per_cta gathered rows, columns
// [col0, col0+seg) with seg bytes.
__global__ void __launch_bounds__(512, 1) tma_kernel(const uint16_t* W, const int* idx, int row_bytes, int seg,
                                                     int rows_per_cta, int ntiles, int stages, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int SB = 16384;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * SB);
  uint64_t* empty = full + stages;
  const int tile = blockIdx.x % ntiles, ksp = blockIdx.x / ntiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 15); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int per = SB / seg;
  const int nst = (rows_per_cta + per - 1) / per;
  const uint8_t* base = reinterpret_cast<const uint8_t*>(W) + static_cast<size_t>(tile) * seg;
  if (warp == 0) {
    for (int s = 0; s < nst; ++s) {
      const int slot = s % stages;
      if (s >= stages) mbar_wait(&empty[slot], ((s / stages) - 1) & 1);
      const int cnt = min(per, rows_per_cta - s * per);
      if (lane == 0) mbar_expect(&full[slot], cnt * seg);
      __syncwarp();
      for (int i = lane; i < cnt; i += 32) {
        const int r = idx[ksp * rows_per_cta + s * per + i];
        bulk(sm + slot * SB + i * seg, base + static_cast<size_t>(r) * row_bytes, seg, &full[slot]);
      }
    }
    return;
  }
  float acc = 0.f;
  const int V = seg / 16;
  for (int s = 0; s < nst; ++s) {
    const int slot = s % stages;
    mbar_wait(&full[slot], (s / stages) & 1);
    const int cnt = min(per, rows_per_cta - s * per);
    for (int f = threadIdx.x - 32; f < cnt * V; f += 480) {
      const uint4 u = *reinterpret_cast<const uint4*>(sm + slot * SB + f * 16);
      acc += __uint_as_float(u.x << 16) + __uint_as_float(u.w);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  if (acc == 12345.f) out[blockIdx.x] = acc;
}

template <int U>
__global__ void __launch_bounds__(512, 1) ldg_kernel(const uint16_t* W, const int* idx, int row_bytes, int seg,
                                                     int rows_per_cta, int ntiles, float* out) {
  const int tile = blockIdx.x % ntiles, ksp = blockIdx.x / ntiles;
  const int V = seg / 16;  // lanes per row segment
  const int rows_per_warp_iter = 32 / V > 0 ? 32 / V : 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / V, v = lane % V;
  const bool ok = sub < rows_per_warp_iter;
  const uint8_t* base = reinterpret_cast<const uint8_t*>(W) + static_cast<size_t>(tile) * seg + v * 16;
  float acc = 0.f;
  const int step = 16 * rows_per_warp_iter;
  for (int r0 = warp * rows_per_warp_iter + sub; r0 < rows_per_cta; r0 += step * U) {
    uint4 u[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int r = r0 + q * step;
      if (ok && r < rows_per_cta) {
        const int row = __ldg(idx + ksp * rows_per_cta + r);
        u[q] = __ldg(reinterpret_cast<const uint4*>(base + static_cast<size_t>(row) * row_bytes));
      } else {
        u[q] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int q = 0; q < U; ++q) acc += __uint_as_float(u[q].x << 16) + __uint_as_float(u[q].w);
  }
  if (acc == 12345.f) out[blockIdx.x] = acc;
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total_rows = 64 * 1024;   // rows of 8 KB = 512 MB (> L2)
  const int row_bytes = 8192;
  uint16_t* W;
  cudaMalloc(&W, total_rows * row_bytes);
  cudaMemset(W, 0, total_rows * row_bytes);
  float* out;
  cudaMalloc(&out, 4096 * 4);
  const int segs[] = {512, 1024, 2048, 4096, 8192};
  printf("kind seg stages/unroll rows_per_cta GB/s us\n");
  for (int seg : segs) {
    const int ntiles = row_bytes / seg;
    const int ks = sms / ntiles > 0 ? sms / ntiles : 1;
    const int grid = ntiles * ks;
    // ~36 MB per launch (a gate_proj-sized sparse linear), rows split over k-splits
    const int rows_total = static_cast<int>((36u << 20) / row_bytes);
    const int rows_per_cta = rows_total / ks;
    std::vector<int> h(ks * rows_per_cta);
    uint32_t st = 12345;
    for (auto& v : h) { st = st * 1664525u + 1013904223u; v = static_cast<int>(st % total_rows); }
    int* idx;
    cudaMalloc(&idx, h.size() * 4);
    cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    const double bytes = static_cast<double>(grid) * rows_per_cta * seg;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int stages : {4, 8, 12}) {
      const size_t smem = stages * 16384 + 256;
      cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (int it = 0; it < 3; ++it) tma_kernel<<<grid, 512, smem>>>(W, idx, row_bytes, seg, rows_per_cta, ntiles, stages, out);
      cudaEventRecord(e0);
      const int reps = 20;
      for (int it = 0; it < reps; ++it) tma_kernel<<<grid, 512, smem>>>(W, idx, row_bytes, seg, rows_per_cta, ntiles, stages, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("tma %5d %2d %5d %8.1f %7.2f\n", seg, stages, rows_per_cta, bytes / (ms / reps * 1e-3) / 1e9, ms / reps * 1e3);
    }
    auto run_ldg = [&](auto kern, int U) {
      for (int it = 0; it < 3; ++it) kern<<<grid, 512>>>(W, idx, row_bytes, seg, rows_per_cta, ntiles, out);
      cudaEventRecord(e0);
      const int reps = 20;
      for (int it = 0; it < reps; ++it) kern<<<grid, 512>>>(W, idx, row_bytes, seg, rows_per_cta, ntiles, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("ldg %5d %2d %5d %8.1f %7.2f\n", seg, U, rows_per_cta, bytes / (ms / reps * 1e-3) / 1e9, ms / reps * 1e3);
    };
    if (seg <= 512) {
      run_ldg(ldg_kernel<4>, 4);
      run_ldg(ldg_kernel<8>, 8);
      run_ldg(ldg_kernel<16>, 16);
    }
    cudaFree(idx);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
