// gather_probe.cu -- which streaming primitive reads GATHERED weight rows
// fastest on B200?  Every launch reads a fresh set of rows (windows rotate
// over a 2 GB buffer, > 15x L2), so the numbers are HBM numbers.
//   A  ldg   : LDG.128 per lane, U rows in flight per warp, grid = tiles x ksplits
//   B  tma   : one thread issues cp.async.bulk of `seg` bytes per row into an
//              smem ring (stages x 16 KB), 15 consumer warps FMA from smem
//   C  flat  : contiguous read of the same byte count (upper bound)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_probe tools/gather_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e));       \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint4 ldg_nc(const void* p) {
  uint4 u;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "l"(p));
  return u;
}
__device__ __forceinline__ void fma8(float (&a)[8], uint4 u, float c) {
  a[0] = fmaf(c, __uint_as_float(u.x << 16), a[0]);
  a[1] = fmaf(c, __uint_as_float(u.x & 0xffff0000u), a[1]);
  a[2] = fmaf(c, __uint_as_float(u.y << 16), a[2]);
  a[3] = fmaf(c, __uint_as_float(u.y & 0xffff0000u), a[3]);
  a[4] = fmaf(c, __uint_as_float(u.z << 16), a[4]);
  a[5] = fmaf(c, __uint_as_float(u.z & 0xffff0000u), a[5]);
  a[6] = fmaf(c, __uint_as_float(u.w << 16), a[6]);
  a[7] = fmaf(c, __uint_as_float(u.w & 0xffff0000u), a[7]);
}

// ---------------------------------------------------------------- A: LDG
// CTA (tile, ks): rows idx[ks*rpc .. +rpc), bytes [tile*seg, +seg) of each.
// A warp covers CW = seg/512 chunks of 512 B per row; rows spread over the
// 16/CW warp groups; U rows in flight per warp.
template <int U>
__global__ void __launch_bounds__(512, 1) ldg_kernel(const uint8_t* W, const int* idx, int row_bytes, int seg,
                                                     int rpc, int ntiles, float* out) {
  const int tile = blockIdx.x % ntiles, ks = blockIdx.x / ntiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cw = seg / 512;          // warps per row (seg multiple of 512, <= 8192)
  const int groups = 16 / cw, g = warp / cw, c = warp % cw;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (g < groups) {
    const int* my = idx + ks * rpc;
    const uint8_t* base = W + static_cast<size_t>(tile) * seg + c * 512 + lane * 16;
    for (int i0 = g; i0 < rpc; i0 += groups * U) {
      uint4 u[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int i = min(i0 + q * groups, rpc - 1);
        u[q] = ldg_nc(base + static_cast<size_t>(my[i]) * row_bytes);
      }
#pragma unroll
      for (int q = 0; q < U; ++q) fma8(acc, u[q], i0 + q * groups < rpc ? 1.0f : 0.f);
    }
  }
  float s = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) s += acc[e];
  if (s == 12345.f) out[blockIdx.x] = s;
}

// ---------------------------------------------------------------- B: TMA bulk ring
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  }
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(512, 1) tma_kernel(const uint8_t* W, const int* idx, int row_bytes, int seg,
                                                     int rpc, int ntiles, int stages, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int SB = 16384;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * SB);
  uint64_t* empty = full + stages;
  const int tile = blockIdx.x % ntiles, ks = blockIdx.x / ntiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 15);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int per = SB / seg;  // rows per slot
  const int nst = (rpc + per - 1) / per;
  const int* my = idx + ks * rpc;
  const uint8_t* base = W + static_cast<size_t>(tile) * seg;
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < nst; ++s) {
        const int slot = s % stages;
        if (s >= stages) mbar_wait(&empty[slot], ((s / stages) - 1) & 1);
        const int cnt = min(per, rpc - s * per);
        mbar_expect(&full[slot], cnt * seg);
        for (int q = 0; q < cnt; ++q)
          bulk(sm + slot * SB + q * seg, base + static_cast<size_t>(my[s * per + q]) * row_bytes, seg, &full[slot]);
      }
    }
    return;
  }
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int ct = threadIdx.x - 32, nct = 480;
  for (int s = 0; s < nst; ++s) {
    const int slot = s % stages;
    mbar_wait(&full[slot], (s / stages) & 1);
    const int cnt = min(per, rpc - s * per);
    const int vecs = cnt * seg / 16;
    for (int v = ct; v < vecs; v += nct) {
      uint4 u = *reinterpret_cast<const uint4*>(sm + slot * SB + v * 16);
      fma8(acc, u, 1.0f);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  float sum = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) sum += acc[e];
  if (sum == 12345.f) out[blockIdx.x] = sum;
}

// ---------------------------------------------------------------- C: flat read
__global__ void __launch_bounds__(512, 2) flat_kernel(const uint4* p, size_t nvec, float* out) {
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < nvec; i += 4 * stride) {
    uint4 a = ldg_nc(p + i), b = ldg_nc(p + i + stride), c = ldg_nc(p + i + 2 * stride), d = ldg_nc(p + i + 3 * stride);
    fma8(acc, a, 1.f); fma8(acc, b, 1.f); fma8(acc, c, 1.f); fma8(acc, d, 1.f);
  }
  for (; i < nvec; i += stride) fma8(acc, ldg_nc(p + i), 1.f);
  float s = 0;
  for (int e = 0; e < 8; ++e) s += acc[e];
  if (s == 12345.f) out[blockIdx.x] = s;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t BUF = size_t(2) << 30;
  uint8_t* W;
  CK(cudaMalloc(&W, BUF));
  CK(cudaMemset(W, 0, BUF));
  float* out;
  CK(cudaMalloc(&out, 4096 * 4));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 40;
  printf("kind row_bytes seg tiles ks param rows/launch MB/launch us/launch GB/s\n");
  for (int row_bytes : {8192, 22016}) {
    const size_t nrows_buf = BUF / row_bytes;
    const int rows = row_bytes == 8192 ? 2048 : 1536;     // ~16 MB / ~33 MB per launch
    const double mb = double(rows) * row_bytes / 1e6;
    // per rep: rows drawn from a fresh window (sorted ascending, like S)
    const size_t win = nrows_buf / reps;
    for (int seg : {512, 1024, 2048, 4096}) {
      if (row_bytes % seg) continue;
      const int ntiles = row_bytes / seg;
      const int ks = sms / ntiles > 0 ? sms / ntiles : 1;
      const int grid = ntiles * ks;
      const int rpc = (rows + ks - 1) / ks;
      std::vector<int> h(size_t(reps) * ks * rpc);
      uint32_t st = 12345;
      for (int r = 0; r < reps; ++r) {
        std::vector<int> pick;
        for (size_t j = 0; j < win && int(pick.size()) < ks * rpc; ++j) {
          st = st * 1664525u + 1013904223u;
          if ((st >> 8) % win < size_t(ks) * rpc * 2) pick.push_back(int(r * win + j));
        }
        while (int(pick.size()) < ks * rpc) pick.push_back(int(r * win));
        for (int i = 0; i < ks * rpc; ++i) h[size_t(r) * ks * rpc + i] = pick[i];
      }
      int* idx;
      CK(cudaMalloc(&idx, h.size() * 4));
      CK(cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
      const double bytes = double(grid) * rpc * seg;
      auto timeit = [&](auto launch) {
        for (int r = 0; r < 3; ++r) launch(r);
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        for (int r = 0; r < reps; ++r) launch(r);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        return ms * 1e3 / reps;
      };
      for (int U : {8, 16}) {
        float us;
        if (U == 8)
          us = timeit([&](int r) {
            ldg_kernel<8><<<grid, 512>>>(W, idx + size_t(r) * ks * rpc, row_bytes, seg, rpc, ntiles, out);
          });
        else
          us = timeit([&](int r) {
            ldg_kernel<16><<<grid, 512>>>(W, idx + size_t(r) * ks * rpc, row_bytes, seg, rpc, ntiles, out);
          });
        printf("ldg %6d %5d %3d %3d U=%-3d %6d %7.2f %7.2f %8.1f\n", row_bytes, seg, ntiles, ks, U, ks * rpc,
               bytes / 1e6, us, bytes / us / 1e3);
      }
      for (int stages : {6, 12}) {
        const size_t smem = stages * 16384 + 256;
        CK(cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        const float us = timeit([&](int r) {
          tma_kernel<<<grid, 512, smem>>>(W, idx + size_t(r) * ks * rpc, row_bytes, seg, rpc, ntiles, stages, out);
        });
        printf("tma %6d %5d %3d %3d st=%-3d %6d %7.2f %7.2f %8.1f\n", row_bytes, seg, ntiles, ks, stages, ks * rpc,
               bytes / 1e6, us, bytes / us / 1e3);
      }
      CK(cudaFree(idx));
    }
    // flat read of the same bytes, rotating windows
    const size_t nvec = size_t(rows) * row_bytes / 16;
    for (int g : {sms, 2 * sms, 4 * sms}) {
      const float us = 0;
      (void)us;
      auto l = [&](int r) {
        flat_kernel<<<g, 512>>>(reinterpret_cast<const uint4*>(W + size_t(r) * ((BUF / reps) & ~size_t(4095))), nvec, out);
      };
      for (int r = 0; r < 3; ++r) l(r);
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      for (int r = 0; r < reps; ++r) l(r);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const float t = ms * 1e3 / reps;
      printf("flat %6d %5d %3d %3d g=%-4d %6d %7.2f %7.2f %8.1f\n", row_bytes, 0, 0, 0, g, rows, mb, t,
             mb * 1e6 / t / 1e3);
    }
  }
  CK(cudaDeviceSynchronize());
  printf("status ok\n");
  return 0;
}
