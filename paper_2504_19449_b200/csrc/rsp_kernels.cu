// rsp_kernels.cu -- sm_100a kernels of the R-Sparse linear operator.
//
// The hot path is ONE persistent kernel per linear (fused_forward_kernel):
//
//   y = W[:, S] x_S  +  A_r (B_r[:, S^c] x_{S^c})        (layer.cpp:95-123)
//
// restated in the input-channel-major form the B200 layout makes cheap:
//
//   t = sum_{j in S^c} x_j * Bt[j, :]         stage 1: gathered rows of B_r^T (length r)
//   y = sum_{j in S}   x_j * Wt[j, :]         gathered rows of W^T (length m)
//     + sum_{c < r}    t_c * At[c, :]         stage 2: rows of A_r^T (length m)
//
// so every term is a gathered-row AXPY over contiguous rows: each row (or its
// column-tile segment) is one cp.async.bulk copy streamed through a shared
// memory ring by a producer warp; 15 consumer warps do fp32 FMAs.
//
// Grid = col_tiles x k_splits CTAs (<= #SMs, one CTA per SM, all co-resident).
// Each CTA redundantly computes the exact top-k selection from x (n <= 64K)
// in shared memory, then takes a balanced rank range of S for its column
// tile, a rank range of S^c for stage 1 and a slice of the r low-rank rows.
// Cross-CTA dependencies use generation barriers in the workspace:
//   * grid barrier: stage-1 partial t vectors -> every CTA (reached early,
//     waited on only after the CTA's W rows are done, so it is hidden);
//   * per-column-tile barrier: split-K partials of y -> deterministic
//     fixed-order reduction (no float atomics: results are bit-reproducible).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "rsp_device.cuh"
#include "rsp_internal.h"

namespace rsp {

// Shared-memory carve-up of the fused kernel (host and device agree).
struct SmemLayout {
  uint32_t off_w, off_u, off_a, off_red, off_misc, off_bar, total;

  __host__ __device__ static uint32_t up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

  __host__ __device__ static SmemLayout make(int stages, int stage_bytes, int n, int cap_w,
                                             int cap_u, int cap_a) {
    SmemLayout L;
    const uint32_t ring = static_cast<uint32_t>(stages) * static_cast<uint32_t>(stage_bytes);
    const uint32_t sel = 4u * static_cast<uint32_t>(n) + 4u * kHistBins;
    uint32_t o = up(ring > sel ? ring : sel, 128);
    L.off_w = o;
    o = up(o + 8u * cap_w, 16);
    L.off_u = o;
    o = up(o + 8u * cap_u, 16);
    L.off_a = o;
    o = up(o + 4u * cap_a, 16);
    L.off_red = o;
    o += kConsumerWarps * 32 * 8 * 4;
    L.off_misc = o;
    o += 128;
    L.off_bar = o;
    o += 16u * stages;
    L.total = up(o, 128);
    return L;
  }
};

size_t fused_smem_bytes(const LaunchPlan& p, int n, int /*elem_bytes*/) {
  return SmemLayout::make(p.stages, p.stage_bytes, n, p.cap_w, p.cap_u, p.cap_a).total;
}

template <typename WT>
__global__ void __launch_bounds__(kThreads, 1) fused_forward_kernel(const FusedParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int VE = Vec<WT>::kElems;
  constexpr int ES = static_cast<int>(sizeof(WT));
  const SmemLayout L = SmemLayout::make(p.stages, p.stage_bytes, p.n, p.cap_w, p.cap_u, p.cap_a);
  uint8_t* ring = smem;
  uint32_t* xk = reinterpret_cast<uint32_t*>(smem);
  uint32_t* hist = xk + p.n;
  int2* list_w = reinterpret_cast<int2*>(smem + L.off_w);  // {channel j, bits of x_j}
  int2* list_u = reinterpret_cast<int2*>(smem + L.off_u);
  float* coef_a = reinterpret_cast<float*>(smem + L.off_a);
  float* red = reinterpret_cast<float*>(smem + L.off_red);
  uint32_t* s_warp = reinterpret_cast<uint32_t*>(smem + L.off_misc);
  uint32_t* scratch = s_warp + 20;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.off_bar);
  uint64_t* empty = full + p.stages;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.x, NB = gridDim.x;
  const int ct = b / p.k_splits, ks = b % p.k_splits;

  // Column tile of this CTA, in units of 8 elements (16 B of bf16).
  const int vm = p.m_pad / 8;
  const int v0 = static_cast<int>(static_cast<long long>(vm) * ct / p.col_tiles);
  const int v1 = static_cast<int>(static_cast<long long>(vm) * (ct + 1) / p.col_tiles);
  const int col0 = v0 * 8, tcw = (v1 - v0) * 8;

  const int k_eff = p.dense ? p.n : p.k;
  const bool has_lr = !p.dense && p.r > 0 && k_eff < p.n;
  const int nu = p.n - k_eff;
  const int wlo = static_cast<int>(static_cast<long long>(k_eff) * ks / p.k_splits);
  const int whi = static_cast<int>(static_cast<long long>(k_eff) * (ks + 1) / p.k_splits);
  const int ulo = has_lr ? static_cast<int>(static_cast<long long>(nu) * b / NB) : 0;
  const int uhi = has_lr ? static_cast<int>(static_cast<long long>(nu) * (b + 1) / NB) : 0;
  const int alo = has_lr ? static_cast<int>(static_cast<long long>(p.r) * ks / p.k_splits) : 0;
  const int ahi = has_lr ? static_cast<int>(static_cast<long long>(p.r) * (ks + 1) / p.k_splits) : 0;
  const int nw = whi - wlo, n1 = uhi - ulo, na = ahi - alo;

  const WT* __restrict__ Wt = static_cast<const WT*>(p.Wt);
  const WT* __restrict__ At = static_cast<const WT*>(p.At);
  const WT* __restrict__ Bt = static_cast<const WT*>(p.Bt);
  const int R1B = p.r_pad * ES;  // stage-1 row bytes
  const int RWB = tcw * ES;      // W / A_r tile-row bytes

  if (tid == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  // The low-rank rows this CTA will stream do not depend on x: start pulling
  // them into L2 now (overlaps the previous kernel's tail under PDL and this
  // kernel's selection otherwise).
  if (warp == 0 && has_lr && RWB > 0) {
    for (int i = lane; i < na; i += 32)
      prefetch_l2_bulk(At + static_cast<size_t>(alo + i) * p.m_pad + col0, RWB);
  }
  if (p.pdl) {
    griddep_wait();
    griddep_launch_dependents();
  }

  // ---- 1. selection (redundant per CTA; x is at most a few tens of KB) ----
  load_x_bits(p.x, p.x_bf16 != 0, p.n, xk);
  __syncthreads();
  const Selection sel = p.dense ? Selection{0u, p.n}
                                : block_select(xk, p.n, p.k, p.x_bf16 != 0, hist, s_warp, scratch);

  // ---- 2. this CTA's row lists (rank ranges of S and of S^c) ----
  {
    const int E = (p.n + kThreads - 1) / kThreads;
    const int j0 = min(p.n, tid * E), j1 = min(p.n, j0 + E);
    uint32_t c = 0;
    for (int j = j0; j < j1; ++j) c += is_selected(abs_key(xk[j]), j, sel);
    uint32_t srank = block_excl_scan(c, s_warp, nullptr);
    uint32_t urank = static_cast<uint32_t>(j0) - srank;
    for (int j = j0; j < j1; ++j) {
      const uint32_t bits = xk[j];
      if (is_selected(abs_key(bits), j, sel)) {
        if (srank >= static_cast<uint32_t>(wlo) && srank < static_cast<uint32_t>(whi))
          list_w[srank - wlo] = make_int2(j, static_cast<int>(bits));
        ++srank;
      } else {
        if (urank >= static_cast<uint32_t>(ulo) && urank < static_cast<uint32_t>(uhi))
          list_u[urank - ulo] = make_int2(j, static_cast<int>(bits));
        ++urank;
      }
    }
  }
  fence_proxy_async_smem();  // generic reads of the x region precede async-proxy ring writes
  __syncthreads();

  const int P1 = R1B > 0 ? p.stage_bytes / R1B : 1;  // stage-1 rows per ring stage
  const int P2 = RWB > 0 ? p.stage_bytes / RWB : 1;  // tile rows per ring stage
  const int stages = p.stages;

  if (warp == 0) {
    // ================= producer: one warp issues every bulk copy =================
    const uint64_t pol = l2_evict_first_policy();
    int s = 0;
    for (int i0 = 0; i0 < n1; i0 += P1, ++s) {
      const int cnt = min(P1, n1 - i0), slot = s % stages;
      if (s >= stages) mbar_wait(&empty[slot], ((s / stages) - 1) & 1);
      if (lane == 0) mbar_arrive_expect_tx(&full[slot], static_cast<uint32_t>(cnt * R1B));
      __syncwarp();
      for (int i = lane; i < cnt; i += 32) {
        const int j = list_u[i0 + i].x;
        bulk_g2s(ring + slot * p.stage_bytes + i * R1B, Bt + static_cast<size_t>(j) * p.r_pad, R1B,
                 &full[slot], pol);
      }
    }
    for (int i0 = 0; i0 < nw; i0 += P2, ++s) {
      const int cnt = min(P2, nw - i0), slot = s % stages;
      if (s >= stages) mbar_wait(&empty[slot], ((s / stages) - 1) & 1);
      if (lane == 0) mbar_arrive_expect_tx(&full[slot], static_cast<uint32_t>(cnt * RWB));
      __syncwarp();
      for (int i = lane; i < cnt; i += 32) {
        const int j = list_w[i0 + i].x;
        bulk_g2s(ring + slot * p.stage_bytes + i * RWB, Wt + static_cast<size_t>(j) * p.m_pad + col0,
                 RWB, &full[slot], pol);
      }
    }
    for (int i0 = 0; i0 < na; i0 += P2, ++s) {
      const int cnt = min(P2, na - i0), slot = s % stages;
      if (s >= stages) mbar_wait(&empty[slot], ((s / stages) - 1) & 1);
      if (lane == 0) mbar_arrive_expect_tx(&full[slot], static_cast<uint32_t>(cnt * RWB));
      __syncwarp();
      for (int i = lane; i < cnt; i += 32) {
        bulk_g2s(ring + slot * p.stage_bytes + i * RWB,
                 At + static_cast<size_t>(alo + i0 + i) * p.m_pad + col0, RWB, &full[slot], pol);
      }
    }
    return;
  }

  // ================= consumers: warps 1..15 =================
  const int cw = warp - 1, ctid = tid - 32;
  int s = 0;
  if (has_lr) {
    // ---- stage 1: partial t over this CTA's slice of S^c ----
    const int V1 = R1B / 16, C1 = (V1 + 31) / 32, G1 = kConsumerWarps / C1;
    const int grp = cw / C1, v = (cw % C1) * 32 + lane;
    const bool vok = grp < G1 && v < V1;
    float acc[VE];
#pragma unroll
    for (int e = 0; e < VE; ++e) acc[e] = 0.f;
    for (int i0 = 0; i0 < n1; i0 += P1, ++s) {
      const int cnt = min(P1, n1 - i0), slot = s % stages;
      mbar_wait(&full[slot], (s / stages) & 1);
      if (vok) {
        const uint8_t* base = ring + slot * p.stage_bytes + v * 16;
        for (int i = grp; i < cnt; i += G1) {
          const float c = __int_as_float(list_u[i0 + i].y);
          Vec<WT>::fma(acc, *reinterpret_cast<const uint4*>(base + i * R1B), c);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
    if (vok) {
#pragma unroll
      for (int e = 0; e < VE; ++e) red[grp * p.r_pad + v * VE + e] = acc[e];
    }
    named_bar_sync(1, kConsumerThreads);
    for (int c = ctid; c < p.r_pad; c += kConsumerThreads) {
      float sum = 0.f;
      for (int g = 0; g < G1; ++g) sum += red[g * p.r_pad + c];
      p.t_part[static_cast<size_t>(b) * p.r_pad + c] = sum;
    }
    __threadfence();
    named_bar_sync(1, kConsumerThreads);
    if (ctid == 0) scratch[4] = gbar_arrive(p.bars, static_cast<unsigned>(NB));
  }

  // ---- gathered W rows (and then A_r rows) of this CTA's column tile ----
  const int V2 = RWB / 16, C2 = (V2 + 31) / 32, G2 = C2 > 0 ? kConsumerWarps / C2 : 0;
  const int grp2 = C2 > 0 ? cw / C2 : 0, v2 = C2 > 0 ? (cw % C2) * 32 + lane : 0;
  const bool vok2 = grp2 < G2 && v2 < V2;
  float acc2[VE];
#pragma unroll
  for (int e = 0; e < VE; ++e) acc2[e] = 0.f;
  for (int i0 = 0; i0 < nw; i0 += P2, ++s) {
    const int cnt = min(P2, nw - i0), slot = s % stages;
    mbar_wait(&full[slot], (s / stages) & 1);
    if (vok2) {
      const uint8_t* base = ring + slot * p.stage_bytes + v2 * 16;
      for (int i = grp2; i < cnt; i += G2) {
        const float c = __int_as_float(list_w[i0 + i].y);
        Vec<WT>::fma(acc2, *reinterpret_cast<const uint4*>(base + i * RWB), c);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  if (has_lr) {
    if (ctid == 0) gbar_wait(p.bars, scratch[4]);
    named_bar_sync(1, kConsumerThreads);
    // t_c for this CTA's low-rank rows: fixed-order sum of the stage-1 partials.
    for (int c = alo + cw; c < ahi; c += kConsumerWarps) {
      float sum = 0.f;
      for (int bb = lane; bb < NB; bb += 32) sum += __ldcg(p.t_part + static_cast<size_t>(bb) * p.r_pad + c);
#pragma unroll
      for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane == 0) coef_a[c - alo] = sum;
    }
    named_bar_sync(1, kConsumerThreads);
    for (int i0 = 0; i0 < na; i0 += P2, ++s) {
      const int cnt = min(P2, na - i0), slot = s % stages;
      mbar_wait(&full[slot], (s / stages) & 1);
      if (vok2) {
        const uint8_t* base = ring + slot * p.stage_bytes + v2 * 16;
        for (int i = grp2; i < cnt; i += G2)
          Vec<WT>::fma(acc2, *reinterpret_cast<const uint4*>(base + i * RWB), coef_a[i0 + i]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
  }

  // ---- split-K: partial tile -> workspace, per-tile barrier, fixed-order sum ----
  if (vok2) {
#pragma unroll
    for (int e = 0; e < VE; ++e) red[grp2 * tcw + v2 * VE + e] = acc2[e];
  }
  named_bar_sync(1, kConsumerThreads);
  for (int c = ctid; c < tcw; c += kConsumerThreads) {
    float sum = 0.f;
    for (int g = 0; g < G2; ++g) sum += red[g * tcw + c];
    p.y_part[static_cast<size_t>(ks) * p.m_pad + col0 + c] = sum;
  }
  __threadfence();
  named_bar_sync(1, kConsumerThreads);
  unsigned* tbar = p.bars + 2 + 2 * ct;
  if (ctid == 0) {
    const unsigned g = gbar_arrive(tbar, static_cast<unsigned>(p.k_splits));
    gbar_wait(tbar, g);
  }
  named_bar_sync(1, kConsumerThreads);
  const int c_lo = static_cast<int>(static_cast<long long>(tcw) * ks / p.k_splits);
  const int c_hi = static_cast<int>(static_cast<long long>(tcw) * (ks + 1) / p.k_splits);
  for (int c = c_lo + ctid; c < c_hi; c += kConsumerThreads) {
    const int col = col0 + c;
    if (col >= p.m) break;
    float sum = 0.f;
#pragma unroll 8
    for (int kk = 0; kk < p.k_splits; ++kk) sum += __ldcg(p.y_part + static_cast<size_t>(kk) * p.m_pad + col);
    p.y[col] = sum;
  }
}

cudaError_t fused_set_smem(int elem_bytes, size_t smem) {
  if (elem_bytes == 2)
    return cudaFuncSetAttribute(fused_forward_kernel<__nv_bfloat16>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  return cudaFuncSetAttribute(fused_forward_kernel<float>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
}

cudaError_t launch_fused(const FusedParams& p, int elem_bytes, int grid, size_t smem,
                         cudaStream_t stream, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  FusedParams q = p;
  q.pdl = pdl ? 1 : 0;
  if (elem_bytes == 2) return cudaLaunchKernelEx(&cfg, fused_forward_kernel<__nv_bfloat16>, q);
  return cudaLaunchKernelEx(&cfg, fused_forward_kernel<float>, q);
}

// ---------------------------------------------------------------------------
// Stand-alone selector (top_k_by_magnitude / threshold_sparsify): one CTA.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1)
    select_kernel(const void* x, int x_bf16, int n, int k, int32_t* kept, int32_t* rest,
                  float* sparse_x) {
  extern __shared__ __align__(16) uint8_t smem_sel[];
  uint32_t* xk = reinterpret_cast<uint32_t*>(smem_sel);
  uint32_t* hist = xk + n;
  uint32_t* s_warp = hist + kHistBins;
  uint32_t* scratch = s_warp + 20;
  load_x_bits(x, x_bf16 != 0, n, xk);
  __syncthreads();
  const Selection sel = block_select(xk, n, k, x_bf16 != 0, hist, s_warp, scratch);
  const int E = (n + kThreads - 1) / kThreads;
  const int j0 = min(n, static_cast<int>(threadIdx.x) * E), j1 = min(n, j0 + E);
  uint32_t c = 0;
  for (int j = j0; j < j1; ++j) c += is_selected(abs_key(xk[j]), j, sel);
  uint32_t srank = block_excl_scan(c, s_warp, nullptr);
  uint32_t urank = static_cast<uint32_t>(j0) - srank;
  for (int j = j0; j < j1; ++j) {
    const uint32_t bits = xk[j];
    const bool in = is_selected(abs_key(bits), j, sel);
    if (in) {
      if (kept) kept[srank] = j;
      ++srank;
    } else {
      if (rest) rest[urank] = j;
      ++urank;
    }
    if (sparse_x) sparse_x[j] = in ? __uint_as_float(bits) : 0.f;
  }
}

size_t select_smem_bytes(int n) { return 4u * static_cast<size_t>(n) + 4u * kHistBins + 256u; }

cudaError_t launch_select(const void* x, bool x_bf16, int n, int k, int32_t* kept, int32_t* rest,
                          float* sparse_x, cudaStream_t stream) {
  const size_t smem = select_smem_bytes(n);
  cudaError_t e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  select_kernel<<<1, kThreads, smem, stream>>>(x, x_bf16 ? 1 : 0, n, k, kept, rest, sparse_x);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// gather_matvec with an explicit kept list (layer.cpp:74-93): one thread per
// output element, kept rows visited in list order.
// ---------------------------------------------------------------------------
template <typename WT>
__device__ __forceinline__ float to_f32(WT v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) {
  return v;
}
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}

template <typename WT>
__global__ void gather_kernel(const WT* __restrict__ Wt, int m, int m_pad, const void* x,
                              int x_bf16, const int32_t* __restrict__ kept, int nkept,
                              float* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  float acc = 0.f;
  for (int t = 0; t < nkept; ++t) {
    const int j = kept[t];
    const float xj = x_bf16 ? __uint_as_float(static_cast<uint32_t>(static_cast<const uint16_t*>(x)[j]) << 16)
                            : static_cast<const float*>(x)[j];
    acc = fmaf(xj, to_f32(Wt[static_cast<size_t>(j) * m_pad + i]), acc);
  }
  y[i] = acc;
}

cudaError_t launch_gather(const void* Wt, int elem_bytes, int m, int m_pad, const void* x,
                          bool x_bf16, const int32_t* kept, int nkept, float* y,
                          cudaStream_t stream) {
  const int threads = 256, blocks = (m + threads - 1) / threads;
  if (m <= 0) return cudaSuccess;
  if (elem_bytes == 2)
    gather_kernel<<<blocks, threads, 0, stream>>>(static_cast<const __nv_bfloat16*>(Wt), m, m_pad,
                                                  x, x_bf16, kept, nkept, y);
  else
    gather_kernel<<<blocks, threads, 0, stream>>>(static_cast<const float*>(Wt), m, m_pad, x,
                                                  x_bf16, kept, nkept, y);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Layout / dtype conversion for device-resident sources (offline; create()).
// f64 is rounded to f32 first and then to bf16 (the same double rounding as
// the host path and as torch's double -> bfloat16).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float src_to_f32(const void* src, int dt, size_t idx) {
  if (dt == 0) return static_cast<const float*>(src)[idx];
  if (dt == 1) return __bfloat162float(static_cast<const __nv_bfloat16*>(src)[idx]);
  return __double2float_rn(static_cast<const double*>(src)[idx]);
}

__global__ void convert_kernel(const void* src, int src_dtype, size_t rows, size_t cols,
                               size_t src_ld, void* dst, int dst_elem, size_t dst_ld,
                               int transpose) {
  __shared__ float tile[32][33];
  const size_t r0 = static_cast<size_t>(blockIdx.y) * 32, c0 = static_cast<size_t>(blockIdx.x) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int dy = ty; dy < 32; dy += 8) {
    const size_t r = r0 + dy, c = c0 + tx;
    if (r < rows && c < cols) tile[dy][tx] = src_to_f32(src, src_dtype, r * src_ld + c);
  }
  __syncthreads();
  for (int dy = ty; dy < 32; dy += 8) {
    size_t dr, dc;
    float v;
    bool ok;
    if (transpose) {
      dr = c0 + dy;
      dc = r0 + tx;
      ok = dr < cols && dc < rows;
      v = tile[tx][dy];
    } else {
      dr = r0 + dy;
      dc = c0 + tx;
      ok = dr < rows && dc < cols;
      v = tile[dy][tx];
    }
    if (!ok) continue;
    if (dst_elem == 4)
      static_cast<float*>(dst)[dr * dst_ld + dc] = v;
    else
      static_cast<__nv_bfloat16*>(dst)[dr * dst_ld + dc] = __float2bfloat16_rn(v);
  }
}

cudaError_t launch_convert(const void* src, int src_dtype, size_t rows, size_t cols, size_t src_ld,
                           void* dst, int dst_elem, size_t dst_ld, bool transpose,
                           cudaStream_t stream) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  const dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  convert_kernel<<<grid, dim3(32, 8), 0, stream>>>(src, src_dtype, rows, cols, src_ld, dst, dst_elem,
                                                   dst_ld, transpose ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace rsp
