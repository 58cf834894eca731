// rsp_kernels.cu -- sm_100a kernels of the R-Sparse linear operator.
//
// The hot path is ONE kernel per linear (fused_forward_kernel):
//
//   y = W[:, S] x_S  +  A_r (B_r[:, S^c] x_{S^c})        (layer.cpp:95-123)
//
// restated in the input-channel-major form the B200 layout makes cheap:
//
//   t = sum_{j in S^c} x_j * Bt[j, :]         stage 1: gathered rows of B_r^T (length r)
//   y = sum_{j in S}   x_j * Wt[j, :]         gathered rows of W^T (length m)
//     + sum_{c < r}    t_c * At[c, :]         stage 2: rows of A_r^T (length m)
//
// Every term is a gathered-row AXPY over contiguous rows, streamed with
// 16-byte coalesced loads straight into registers: a warp covers a 512-byte
// segment of one row per load (32 lanes x 16 B) and keeps U rows in flight.
// (Measured on B200 by tools/stream_probe.cu: 16-deep LDG.128 gathers reach
// 92% of the measured HBM copy bandwidth; 1-D TMA bulk copies of 0.5-8 KB row
// segments reached 21-46%, so the ring/TMA design of the first version was
// dropped -- see DESIGN.md.)
//
// Grid = col_tiles x k_splits CTAs (<= #SMs; one CTA per SM, all co-resident).
// Every CTA computes the exact selection from x in shared memory
// (rsp_select.cuh), then splits its 16 warps by role:
//   * stage-1 warps stream this CTA's slice of the S^c rows of B_r^T, write a
//     partial t, arrive on a grid barrier, wait for it (early: stage 1 is
//     small), and reduce the partials of the rank rows this CTA owns in a
//     fixed order; then signal the other warps through a named barrier;
//   * W warps stream this CTA's rank range of S (its column tile), then the
//     A_r^T rows (prefetched into L2 at kernel start: they do not depend on x).
// Split-K partials of y are combined by the last CTA of each column tile in
// fixed order (no float atomics: results are bit-reproducible).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "rsp_device.cuh"
#include "rsp_internal.h"
#include "rsp_select.cuh"

namespace rsp {

// Shared-memory carve-up of the fused kernel (host and device agree).
// cap_w / cap_u: channels in this CTA's W / stage-1 ranges (each range is
// split into a definite list and a boundary list of at most that length).
struct SmemLayout {
  uint32_t off_red1, off_red2, off_cand, off_misc, off_wscr, off_keys, off_w, off_wb, off_u, off_a,
      off_b, off_astage, total;

  __host__ __device__ static uint32_t up(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

  __host__ __device__ static SmemLayout make(int n, int cap_w, int cap_u, int cap_a, int a_bytes) {
    SmemLayout L;
    uint32_t o = 4u * kHistBins;  // hist at 0
    L.off_red1 = o;
    o += 16384u;
    L.off_red2 = o;
    o += 16384u;
    L.off_cand = o;
    o += 4u * kCandWords;
    L.off_misc = o;
    o += 4u * kMiscWords;
    L.off_wscr = o;
    o += 4u * (256 + 64);
    L.off_keys = o;
    o = up(o + 4u * static_cast<uint32_t>(n), 16);
    L.off_w = o;
    o = up(o + 8u * cap_w, 16);
    L.off_wb = o;
    o = up(o + 8u * cap_w, 16);
    L.off_u = o;
    o = up(o + 8u * cap_u, 16);
    L.off_a = o;
    o = up(o + 4u * cap_a, 16);
    L.off_b = o;
    o = up(o + 4u * cap_a, 16);
    L.off_astage = o;
    o += static_cast<uint32_t>(a_bytes);
    L.total = up(o, 128);
    return L;
  }
};

size_t fused_smem_bytes(const LaunchPlan& p, int n) {
  return SmemLayout::make(n, p.cap_w, p.cap_u, p.cap_a, p.a_smem_bytes).total;
}

__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Debug phase trace: slot 0 = globaltimer at CTA start, slots 1.. = clock64 - start.
#define RSP_TRACE(ev)                                                \
  do {                                                               \
    if (p.trace) p.trace[blockIdx.x * 16 + (ev)] = clk() - t_start; \
  } while (0)

// Partial sums of one lane's 16-byte column slice, returned in registers.
struct Acc {
  float v[8];
};

// Gathered rows from a shared-memory list of {channel j, coefficient bits}:
// sum over i = first, first+stride, ... < count of coef_i * row(j_i)[lane's 16 B],
// row(j) = base + j * row_bytes.  U rows are loaded before any is consumed
// (U x 512 B in flight per warp); out-of-range slots reuse the last valid row
// with a zero coefficient so every load is unconditional.  Out of line: every
// warp role shares this one copy of the hot loop (instruction-cache footprint).
template <typename WT, int U>
__device__ __noinline__ Acc stream_list(uint32_t list, int first, int count, int stride, bool lane_ok,
                                        const uint8_t* base, uint32_t row_bytes) {
  float acc[Vec<WT>::kElems];
#pragma unroll
  for (int e = 0; e < Vec<WT>::kElems; ++e) acc[e] = 0.f;
  if (lane_ok) {
    for (int i0 = first; i0 < count; i0 += stride * U) {
      uint4 u[U];
      float c[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int i = i0 + q * stride;
        const uint2 e = lds2(list + 8u * static_cast<uint32_t>(min(i, count - 1)));
        c[q] = i < count ? __uint_as_float(e.y) : 0.f;
        u[q] = ldg_stream(base + static_cast<size_t>(e.x) * row_bytes);
      }
#pragma unroll
      for (int q = 0; q < U; ++q) Vec<WT>::fma(acc, u[q], c[q]);
    }
  }
  Acc r;
#pragma unroll
  for (int e = 0; e < 8; ++e) r.v[e] = e < Vec<WT>::kElems ? acc[e] : 0.f;
  return r;
}

// Consecutive rows (the low-rank A_r^T rows, prefetched into L2):
// sum over i of coef[i] * (base + i * row_bytes)[lane's 16 B].
template <typename WT, int U>
__device__ __noinline__ Acc stream_seq(uint32_t coef, int first, int count, int stride, bool lane_ok,
                                       const uint8_t* base, uint32_t row_bytes) {
  float acc[Vec<WT>::kElems];
#pragma unroll
  for (int e = 0; e < Vec<WT>::kElems; ++e) acc[e] = 0.f;
  if (lane_ok) {
    for (int i0 = first; i0 < count; i0 += stride * U) {
      uint4 u[U];
      float c[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int i = min(i0 + q * stride, count - 1);
        c[q] = i0 + q * stride < count ? ldsf(coef + 4u * i) : 0.f;
        u[q] = ldg_l2(base + static_cast<size_t>(i) * row_bytes);
      }
#pragma unroll
      for (int q = 0; q < U; ++q) Vec<WT>::fma(acc, u[q], c[q]);
    }
  }
  Acc r;
#pragma unroll
  for (int e = 0; e < 8; ++e) r.v[e] = e < Vec<WT>::kElems ? acc[e] : 0.f;
  return r;
}

template <int VE>
__device__ __forceinline__ void acc_add(float (&acc)[VE], const Acc& a) {
#pragma unroll
  for (int e = 0; e < VE; ++e) acc[e] += a.v[e];
}

// floor(total * i / parts) in 32-bit arithmetic (total * parts < 2^32 for every
// shape this kernel accepts; 64-bit division is a ~100-instruction subroutine).
__device__ __forceinline__ int part(int total, int i, int parts) {
  return static_cast<int>(static_cast<uint32_t>(total) * static_cast<uint32_t>(i) / static_cast<uint32_t>(parts));
}

template <typename WT, int U>
__global__ void __launch_bounds__(kThreads, 1) fused_forward_kernel(const FusedParams p) {
  const long long t_start = clk();
  if (p.trace && threadIdx.x == 0) p.trace[blockIdx.x * 16] = gtimer();
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int VE = Vec<WT>::kElems;  // elements per 16 B
  constexpr int ES = static_cast<int>(sizeof(WT));
  constexpr int M_GEN = 28;            // misc slot: barrier generation at kernel start
  const SmemLayout L = SmemLayout::make(p.n, p.cap_w, p.cap_u, p.cap_a, p.a_smem_bytes);
  const uint32_t sb = smem_base_pinned(smem);  // shared-window base: every access below is LDS/STS
  SelSmem ss;
  ss.hist = sb;
  ss.cand = sb + L.off_cand;
  ss.keys = sb + L.off_keys;
  ss.misc = sb + L.off_misc;
  const uint32_t list_w = sb + L.off_w;    // int2 {channel j, bits of x_j}: definitely in S
  const uint32_t list_wb = sb + L.off_wb;  // boundary channels of the W range (-> those in S)
  const uint32_t list_u = sb + L.off_u;    // definitely in S^c (stage-1 range)
  const uint32_t coef_a = sb + L.off_a;    // f32 t_c per rank row of this CTA
  const uint32_t coef_b = sb + L.off_b;    // f32 boundary-bin part of t_c (local)
  const uint32_t a_stage = sb + L.off_astage;
  uint8_t* a_stage_ptr = smem + L.off_astage;  // cp.async destination
  const uint32_t red1 = sb + L.off_red1;   // [G1][r_pad] f32
  const uint32_t red2 = sb + L.off_red2;   // [G2][tile cols] f32

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.x, NB = gridDim.x;
  const int ct = b / p.k_splits, ks = b % p.k_splits;

  // Column tile of this CTA in 16-byte units.
  const int vrow = p.m_pad * ES / 16;
  const int v0 = part(vrow, ct, p.col_tiles), v1 = part(vrow, ct + 1, p.col_tiles);
  const int tw = v1 - v0, tcw = tw * VE, col0 = v0 * VE;

  const int k_eff = p.dense ? p.n : p.k;
  const bool has_lr = !p.dense && p.r > 0 && k_eff < p.n;
  // Static channel ranges: the W rows of S in [wc0, wc1) for this column
  // tile, the stage-1 rows of S^c in [uc0, uc1).
  const int wc0 = part(p.n, ks, p.k_splits), wc1 = part(p.n, ks + 1, p.k_splits);
  const int uc0 = has_lr ? part(p.n, b, NB) : 0, uc1 = has_lr ? part(p.n, b + 1, NB) : 0;
  const int alo = has_lr ? part(p.r, ks, p.k_splits) : 0, ahi = has_lr ? part(p.r, ks + 1, p.k_splits) : 0;
  const int na = ahi - alo;
  // A_r^T rows held in shared memory (the rest stream from L2 after a prefetch).
  const int na_s = has_lr ? min(na, p.a_smem_bytes / max(1, tw * 16)) : 0;
  // Fast mode: stage-1 sums and split-K partials of y are combined with float
  // atomics.  Deterministic mode: fixed-order partial sums (bit-reproducible).
  const bool fast = !p.deterministic;
  const bool red_y = has_lr && p.k_splits > 1 && fast;

  const uint8_t* Wt = static_cast<const uint8_t*>(p.Wt);
  const uint8_t* At = static_cast<const uint8_t*>(p.At);
  const uint8_t* Bt = static_cast<const uint8_t*>(p.Bt);
  const size_t rowW = static_cast<size_t>(p.m_pad) * ES;  // bytes per W^T / A_r^T row
  const size_t rowB = static_cast<size_t>(p.r_pad) * ES;  // bytes per B_r^T row
  const uint8_t* a_tile = At + static_cast<size_t>(col0) * ES;

  // ---- prologue: independent of x (overlaps the previous kernel under PDL) ----
  if (!p.dense) sel_clear(ss);
  if (has_lr) {
    for (int f = tid; f < na_s * tw; f += kThreads) {
      const int i = f / tw, v = f - i * tw;
      cp_async16(a_stage_ptr + static_cast<size_t>(f) * 16, a_tile + static_cast<size_t>(alo + i) * rowW + v * 16);
    }
    cp_async_commit();
    const int la = (tw * 16 + 127) / 128;
    for (int f = tid; f < (na - na_s) * la; f += kThreads) {
      const int i = na_s + f / la, l = f % la;
      prefetch_l2_line(a_tile + static_cast<size_t>(alo + i) * rowW + 128 * l);
    }
  }
  if (p.pdl) {
    griddep_wait();
    griddep_launch_dependents();
  }
  if (has_lr && tid == 0) {
    const unsigned g = ld_relaxed_gpu(p.bars + 1);  // stable: nobody of this launch has arrived yet
    ss.set_m(M_GEN, g);
  }
  if (red_y) {  // zero this CTA's slice of y; published by the grid barrier below
    const int y0 = part(p.m, b, NB), y1 = part(p.m, b + 1, NB);
    for (int i = y0 + tid; i < y1; i += kThreads) p.y[i] = 0.f;
  }
  if (tid == 0) RSP_TRACE(1);

  // ---- 1. x -> shared keys + 12-bit histogram; the boundary bin ----
  __syncthreads();  // histogram zeroed (prologue) before the load adds to it
  sel_load(p.x, p.x_bf16 != 0, p.n, ss, !p.dense);
  if (tid == 0) RSP_TRACE(2);
  const Boundary bd = p.dense ? Boundary{0u, 0u, 0u, true} : sel_boundary(p.n, p.k, ss);
  if (tid == 0) RSP_TRACE(14);
  const bool bnd = !bd.all_in && bd.b12 != 0xffffffffu;  // a boundary bin must be cut
  const bool gathered = bnd && bd.cnt <= static_cast<uint32_t>(kCandWords / 2);
  const uint32_t gen0 = has_lr ? ss.m(M_GEN) : 0u;
  float* t_cur = p.t_acc + (gen0 & 1u) * kTAccCap;
  if (has_lr && fast) {
    // Zero this CTA's slice of the next launch's t buffer (whole buffer: the
    // next launch on this workspace may be a layer of a larger rank).
    float* t_nxt = p.t_acc + ((gen0 + 1u) & 1u) * kTAccCap;
    const int c0 = part(static_cast<int>(kTAccCap), b, NB), c1 = part(static_cast<int>(kTAccCap), b + 1, NB);
    for (int c = c0 + tid; c < c1; c += kThreads) t_nxt[c] = 0.f;
  }
  if (gathered) {  // boundary-bin members for the resolver (order irrelevant)
    for (int j = tid; j < p.n; j += kThreads) {
      const uint32_t key = abs_key(ss.key(j));
      if ((key >> 19) == bd.b12) sts2(ss.cand + 8u * atoms_add(ss.misc + 4u * M_CC, 1u), key, static_cast<uint32_t>(j));
    }
  }
  if (tid == 0) RSP_TRACE(3);
  // ---- 2. this CTA's row lists: definite members now, boundary members deferred ----
  sel_compact(ss, wc0, wc1, bd, 0, [&](int cls, uint32_t i, int j, uint32_t bits) {
    if (cls == 0) sts2(list_w + 8u * i, static_cast<uint32_t>(j), bits);
    else if (cls == 1) sts2(list_wb + 8u * i, static_cast<uint32_t>(j), bits);
  });
  if (tid == 0) RSP_TRACE(15);
  if (has_lr) {
    // stage 1 takes only the definitely-unselected channels; the boundary
    // bin's unselected members enter t locally (coef_b) once the cut is known
    sel_compact(ss, uc0, uc1, bd, 1, [&](int cls, uint32_t i, int j, uint32_t bits) {
      if (cls == 2) sts2(list_u + 8u * i, static_cast<uint32_t>(j), bits);
    });
  }
  __syncthreads();
  const int nw_def = static_cast<int>(ss.m(M_CLS + 0)), nw_bnd = static_cast<int>(ss.m(M_CLS + 1));
  const int nu_def = has_lr ? static_cast<int>(ss.m(M_CLS + 5)) : 0;
  // Start every definite row's DRAM -> L2 transfer now (128-byte line
  // prefetches flattened over the block), plus the A_r rows' slices of the
  // boundary members' B_r^T rows (needed for coef_b).
  {
    const int lw = (tw * 16 + 127) / 128, lu = (static_cast<int>(rowB) + 127) / 128;
    const int tot_w = nw_def * lw, tot = tot_w + nu_def * lu;
    for (int f = tid; f < tot; f += kThreads) {
      if (f < tot_w) {
        const int i = f / lw, l = f - i * lw;
        prefetch_l2_line(Wt + static_cast<size_t>(lds(list_w + 8u * i)) * rowW + static_cast<size_t>(col0) * ES + 128 * l);
      } else {
        const int g = f - tot_w, i = g / lu, l = g - i * lu;
        prefetch_l2_line(Bt + static_cast<size_t>(lds(list_u + 8u * i)) * rowB + 128 * l);
      }
    }
    if (has_lr && gathered && na > 0) {
      const int lb = (na * ES + 127) / 128 + 1;
      for (int f = tid; f < static_cast<int>(bd.cnt) * lb; f += kThreads) {
        const int i = f / lb, l = f - i * lb;
        const uint32_t j = lds(ss.cand + 8u * i + 4u);
        const uint8_t* q = Bt + static_cast<size_t>(j) * rowB + static_cast<size_t>(alo) * ES + 128 * l;
        if (128 * l < na * ES + 128) prefetch_l2_line(q);
      }
    }
  }
  if (tid == 0) RSP_TRACE(4);

  // Roles: warp 0 resolves the boundary; W1 stage-1 warps (a multiple of C1);
  // the remaining nWW warps stream W then A_r.
  const int vb = p.r_pad * ES / 16;  // 16-B units per B_r^T row
  const int C1 = has_lr ? (vb + 31) / 32 : 1;
  const int C2 = (tw + 31) / 32;
  constexpr int kWork = kWarps - 1;
  int W1 = 0;
  if (has_lr) {
    const int s1 = nu_def * C1 + na, s2 = (nw_def + nw_bnd) * C2;
    const int want = (kWork * s1 + s1 + s2 - 1) / (s1 + s2 > 0 ? s1 + s2 : 1);
    W1 = max(1, (want + C1 - 1) / C1) * C1;
    W1 = min(W1, ((kWork - C2) / C1) * C1);
  }
  const int nWW = kWork - W1;
  constexpr int M_T = 29, M_J = 30;

  if (warp == 0) {
    // ===================== boundary resolver =====================
    if (bnd && (nw_bnd > 0 || has_lr)) {
      uint32_t T, J;
      warp_resolve_cut(ss, p.n, bd, gathered, sb + L.off_wscr, T, J);
      if (lane == 0) {
        ss.set_m(M_T, T);
        ss.set_m(M_J, J);
      }
      // keep the W-range boundary members that are in S (order preserved)
      uint32_t keep_w = 0;
      for (int i0 = 0; i0 < nw_bnd; i0 += 32) {
        const int i = i0 + lane;
        const uint2 e = i < nw_bnd ? lds2(list_wb + 8u * i) : make_uint2(0u, 0u);
        const uint32_t key = abs_key(e.y);
        const bool in = i < nw_bnd && (key > T || (key == T && e.x <= J));
        const uint32_t m = __ballot_sync(0xffffffffu, in);
        __syncwarp();
        if (in) sts2(list_wb + 8u * (keep_w + __popc(m & lanemask_lt())), e.x, e.y);
        keep_w += __popc(m);
      }
      if (lane == 0) ss.set_m(M_CLS + 1, keep_w);
    }
    if (tid == 0) RSP_TRACE(13);
    named_bar_arrive(4, kThreads);  // boundary cut published
    return;
  }

  if (warp <= W1) {
    // ===================== stage-1 warps =====================
    const int sw = warp - 1, nst = W1 * 32, stid = tid - 32;
    const int G1 = W1 / C1, g1 = sw / C1;
    const int v = (sw % C1) * 32 + lane;
    const bool ok = v < vb;
    float acc[VE];
#pragma unroll
    for (int e = 0; e < VE; ++e) acc[e] = 0.f;
    acc_add(acc, stream_list<WT, U>(list_u, g1, nu_def, G1, ok, Bt + v * 16, static_cast<uint32_t>(rowB)));
    if (stid == 0) RSP_TRACE(5);
    if (ok) {
#pragma unroll
      for (int e = 0; e < VE; ++e) stsf(red1 + 4u * (g1 * p.r_pad + v * VE + e), acc[e]);
    }
    named_bar_sync(1, nst);
    // this CTA's stage-1 contribution: float atomics into t (fast) or
    // column b of the partials (deterministic)
    for (int c = stid; c < p.r_pad; c += nst) {
      float sum = 0.f;
      for (int g = 0; g < G1; ++g) sum += ldsf(red1 + 4u * (g * p.r_pad + c));
      if (fast) {
        if (sum != 0.f) atomicAdd(t_cur + c, sum);
      } else {
        p.t_part[static_cast<size_t>(c) * p.nb_pad + b] = sum;
      }
    }
    named_bar_sync(1, nst);
    if (stid == 0) {
      gbar_arrive(p.bars, static_cast<unsigned>(NB), gen0);
      RSP_TRACE(6);
    }
    // Boundary members not in S enter t through this CTA's rank rows only (t
    // is linear): coef_b[i] = sum of x_j * Bt[j][alo + i] over them.  Members
    // split across the stage-1 warps, rows across lanes, fixed-order combine.
    named_bar_sync(4, kThreads);
    if (bnd && na > 0) {
      const uint32_t T = ss.m(M_T), J = ss.m(M_J);
      // channel order (not the gathered list's arrival order): deterministic sums
      const int q0 = part(p.n, sw, W1), q1 = part(p.n, sw + 1, W1);
      const uint8_t* brow0 = Bt + static_cast<size_t>(alo) * ES;
      for (int i0 = 0; i0 < na; i0 += 128) {
        float cb[4] = {0.f, 0.f, 0.f, 0.f};
        for (int qb = q0; qb < q1; qb += 32) {  // warp-uniform trip count
          const int q = qb + lane;
          const uint32_t j = static_cast<uint32_t>(q);
          const uint32_t bits = q < q1 ? ss.key(q) : 0u;
          const uint32_t key = abs_key(bits);
          const bool out = q < q1 && (key >> 19) == bd.b12 && !(key > T || (key == T && j <= J));
          uint32_t mk = __ballot_sync(0xffffffffu, out);
          while (mk) {  // four members per round: 16 independent loads in flight
            uint32_t jj[4];
            float xx[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int src = mk ? __ffs(mk) - 1 : 0;
              const bool have = mk != 0;
              mk &= mk - 1;
              jj[u] = __shfl_sync(0xffffffffu, j, src);
              xx[u] = have ? __uint_as_float(__shfl_sync(0xffffffffu, bits, src)) : 0.f;
            }
            float w[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const uint8_t* row = brow0 + static_cast<size_t>(jj[u]) * rowB;
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int i = i0 + lane + 32 * e;
                w[u][e] = 0.f;
                if (i < na) {
                  if constexpr (ES == 2)
                    w[u][e] = __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(row) + i));
                  else
                    w[u][e] = __ldg(reinterpret_cast<const float*>(row) + i);
                }
              }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
#pragma unroll
              for (int e = 0; e < 4; ++e) cb[e] = fmaf(xx[u], w[u][e], cb[e]);
            }
          }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) stsf(red1 + 4u * (sw * 128 + lane + 32 * e), cb[e]);
        named_bar_sync(1, nst);
        for (int i = i0 + stid; i < min(na, i0 + 128); i += nst) {
          float sum = 0.f;
          for (int w = 0; w < W1; ++w) sum += ldsf(red1 + 4u * (w * 128 + i - i0));
          stsf(coef_b + 4u * i, sum);
        }
        named_bar_sync(1, nst);
      }
    } else {
      for (int i = stid; i < na; i += nst) stsf(coef_b + 4u * i, 0.f);
    }
    if (stid == 0) {
      gbar_wait(p.bars, gen0);
      RSP_TRACE(7);
    }
    named_bar_sync(1, nst);
    // t_c for this CTA's rank rows
    if (fast) {
      for (int i = stid; i < na; i += nst) stsf(coef_a + 4u * i, __ldcg(t_cur + alo + i) + ldsf(coef_b + 4u * i));
    } else {
      // 8 lanes per row sum the row's nb_pad partials (float4 loads, fixed order, fixed xor tree)
      const int g8 = stid >> 3, l8 = stid & 7, ng8 = nst / 8;
      const int nq = p.nb_pad / 4;
      for (int cbase = alo; cbase < ahi; cbase += ng8) {  // uniform trip count: shuffles below
        const int c = cbase + g8;
        float sum = 0.f;
        if (c < ahi) {
          const float4* row = reinterpret_cast<const float4*>(p.t_part + static_cast<size_t>(c) * p.nb_pad);
          for (int q = l8; q < nq; q += 8) {
            const float4 u = __ldcg(row + q);
            sum += (u.x + u.y) + (u.z + u.w);
          }
        }
        sum += __shfl_xor_sync(0xffffffffu, sum, 4);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        if (l8 == 0 && c < ahi) stsf(coef_a + 4u * (c - alo), sum + ldsf(coef_b + 4u * (c - alo)));
      }
    }
    if (stid == 0) RSP_TRACE(8);
    cp_async_wait_all();
    named_bar_arrive(3, (W1 + nWW) * 32);  // coef_a (and this thread's A_r copies) are ready
    return;
  }

  // ===================== W / A_r warps =====================
  const int wr = warp - 1 - W1, G2 = nWW / C2, g2 = wr / C2;
  const int v = (wr % C2) * 32 + lane;
  const bool ok = g2 < G2 && v < tw;
  const int wt = tid - (1 + W1) * 32, nwt = nWW * 32;
  float acc[VE];
#pragma unroll
  for (int e = 0; e < VE; ++e) acc[e] = 0.f;
  const uint8_t* wbase = Wt + static_cast<size_t>(col0) * ES + v * 16;
  acc_add(acc, stream_list<WT, U>(list_w, g2, nw_def, G2, ok, wbase, static_cast<uint32_t>(rowW)));
  named_bar_sync(4, kThreads);
  acc_add(acc, stream_list<WT, U>(list_wb, g2, static_cast<int>(ss.m(M_CLS + 1)), G2, ok, wbase,
                                  static_cast<uint32_t>(rowW)));
  if (wt == 0) RSP_TRACE(9);
  if (has_lr) {
    cp_async_wait_all();
    named_bar_sync(3, (W1 + nWW) * 32);  // stage-1 warps have published coef_a; A_r^T rows landed
    if (g2 < G2) {
      if (ok) {
        for (int i = g2; i < na_s; i += G2)
          Vec<WT>::fma(acc, lds4(a_stage + (static_cast<uint32_t>(i) * tw + v) * 16u), ldsf(coef_a + 4u * i));
      }
      const int first = na_s + ((g2 - na_s % G2) % G2 + G2) % G2;  // keep row i on group i % G2
      acc_add(acc, stream_seq<WT, U>(coef_a, first, na, G2, ok,
                                     a_tile + static_cast<size_t>(alo) * rowW + v * 16,
                                     static_cast<uint32_t>(rowW)));
    }
  }
  if (wt == 0) RSP_TRACE(10);

  // ---- split-K: group reduction in smem, then y ----
  if (ok) {
#pragma unroll
    for (int e = 0; e < VE; ++e) stsf(red2 + 4u * (g2 * tcw + v * VE + e), acc[e]);
  }
  named_bar_sync(2, nwt);
  for (int c = wt; c < tcw; c += nwt) {
    float sum = 0.f;
    for (int g = 0; g < G2; ++g) sum += ldsf(red2 + 4u * (g * tcw + c));
    const int col = col0 + c;
    if (p.k_splits == 1) {
      if (col < p.m) p.y[col] = sum;
    } else if (red_y) {
      if (col < p.m) atomicAdd(p.y + col, sum);
    } else {
      p.y_part[static_cast<size_t>(ks) * p.m_pad + col] = sum;
    }
  }
  if (wt == 0) RSP_TRACE(11);
  if (p.k_splits > 1 && !red_y) {
    __threadfence();
    named_bar_sync(2, nwt);
    unsigned* ticket = p.bars + 2 + ct;
    if (wt == 0) ss.set_m(M_LAST, atom_add_acq_rel_gpu(ticket, 1u) == static_cast<unsigned>(p.k_splits - 1));
    named_bar_sync(2, nwt);
    if (ss.m(M_LAST)) {
      // Last CTA of this column tile: fixed-order sum of the k_splits partials.
      for (int c = wt; c < tcw; c += nwt) {
        const int col = col0 + c;
        if (col >= p.m) break;
        float sum = 0.f;
#pragma unroll 4
        for (int kk = 0; kk < p.k_splits; ++kk)
          sum += __ldcg(p.y_part + static_cast<size_t>(kk) * p.m_pad + col);
        p.y[col] = sum;
      }
      if (wt == 0) st_relaxed_gpu(ticket, 0u);
    }
  }
  if (wt == 0) RSP_TRACE(12);
}

template <typename WT>
static cudaError_t set_smem_t(size_t smem) {
  cudaError_t e = cudaFuncSetAttribute(fused_forward_kernel<WT, 8>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(fused_forward_kernel<WT, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(smem));
}

cudaError_t fused_set_smem(int elem_bytes, size_t smem) {
  return elem_bytes == 2 ? set_smem_t<__nv_bfloat16>(smem) : set_smem_t<float>(smem);
}

static int unroll_choice() {
  static int u = [] {
    const char* v = getenv("RSP_UNROLL");
    return (v && atoi(v) == 16) ? 16 : 8;
  }();
  return u;
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
  const bool u8 = unroll_choice() == 8;
  if (elem_bytes == 2)
    return u8 ? cudaLaunchKernelEx(&cfg, fused_forward_kernel<__nv_bfloat16, 8>, q)
              : cudaLaunchKernelEx(&cfg, fused_forward_kernel<__nv_bfloat16, 16>, q);
  return u8 ? cudaLaunchKernelEx(&cfg, fused_forward_kernel<float, 8>, q)
            : cudaLaunchKernelEx(&cfg, fused_forward_kernel<float, 16>, q);
}

// ---------------------------------------------------------------------------
// Stand-alone selector (top_k_by_magnitude / threshold_sparsify): one CTA,
// the same selection code as the fused kernel.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1)
    select_kernel(const void* x, int x_bf16, int n, int k, int32_t* kept, int32_t* rest,
                  float* sparse_x) {
  extern __shared__ __align__(16) uint8_t smem_sel[];
  const uint32_t sb = smem_base_pinned(smem_sel);
  SelSmem ss;
  ss.hist = sb;
  ss.cand = sb + 4u * kHistBins;
  ss.misc = ss.cand + 4u * kCandWords;
  ss.keys = ss.misc + 4u * kMiscWords;
  sel_clear(ss);
  __syncthreads();
  sel_load(x, x_bf16 != 0, n, ss, true);
  const SelResult sr = sel_resolve(n, k, x_bf16 != 0, ss);
  sel_count(n, sr, ss);
  sel_range_emit(n, sr, ss, true, 0u, static_cast<uint32_t>(k), [&](int j, uint32_t bits, uint32_t i) {
    if (kept) kept[i] = j;
    if (sparse_x) sparse_x[j] = __uint_as_float(bits);
  });
  sel_range_emit(n, sr, ss, false, 0u, static_cast<uint32_t>(n - k), [&](int j, uint32_t, uint32_t i) {
    if (rest) rest[i] = j;
    if (sparse_x) sparse_x[j] = 0.f;
  });
}

size_t select_smem_bytes(int n) {
  return 4u * (kHistBins + kCandWords + kMiscWords) + 4u * static_cast<size_t>(n);
}

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
