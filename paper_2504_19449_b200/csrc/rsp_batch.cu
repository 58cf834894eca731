// rsp_batch.cu -- the batch > 1 forward of one R-Sparse linear (config 3,
// SURVEY §8(f)#1), bf16 weights and activations.
//
// Reference semantics: B independent `forward` calls (SPEC.md:325,
// layer.cpp:95-123): token b keeps its own top-k set S_b.  Restated for one
// pass over the weights:
//
//   U      = union of the S_b                     (W rows read once per batch)
//   Y[b]   = sum_{j in U} [j in S_b] x_bj W[:, j]  +  A_r t_b
//   t_b    = sum_{j not in S_b} x_bj B_r[:, j]
//
// Every product is a gathered-row contraction with per-token coefficients,
// run on the tensor cores (mma.sync m16n8k16 bf16 -> fp32; the 16 tokens are
// the M dimension, output columns N, channels K): each warp loads 16 rows x
// 64 columns per step with 16-byte loads (4 steps in flight), stages them
// through a swizzled shared tile and feeds ldmatrix.trans -> mma.  At <= 16
// FLOP/byte the op stays HBM-bound; the tensor cores only keep the issue rate
// (8 x 16 FMAs per 16-byte load on CUDA cores) off the critical path.
//
// Kernels:
//   batch_cut_kernel      one CTA per token: the exact cut (T, jlim) of token b
//                         (the same selector as the batch-1 path);
//   batch_forward_kernel  grid = column tiles x channel splits (<= #SMs, one
//                         CTA per SM): lists of U and of each token's
//                         complement, stage 1 into an L2 t accumulator, a
//                         counting barrier, W rows, stage 2, combine.
#include <algorithm>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "rsp_device.cuh"
#include "rsp_internal.h"
#include "rsp_select.cuh"

namespace rsp {

namespace {

constexpr int kColsPerWarp = 64;  // 8 n-blocks of the m16n8k16 product
constexpr int kStage = 16;        // rows per mma step (K)
constexpr int kDepth = 4;         // steps in flight per warp
constexpr int kRing = 4;          // CTA-cooperative stages (cw == 8)
constexpr int kRingT = 8;         // tcgen05 ring stages (refill lags the MMAs by two steps)

__device__ __forceinline__ int bpart(int total, int i, int parts) {
  return static_cast<int>(static_cast<uint32_t>(total) * static_cast<uint32_t>(i) / static_cast<uint32_t>(parts));
}

__device__ __forceinline__ void ldsm_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr)
               : "memory");
}

__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(uint32_t lo, uint32_t hi) { return (lo & 0xffffu) | (hi << 16); }

// One warp's accumulator: 16 tokens x 64 columns (n-block q: token g / g+8,
// columns 8q + 2t, 8q + 2t + 1 with g = lane / 4, t = lane % 4).
struct Frag {
  float d[8][4];
};

// A step: rows kk = 0..15 of a 16 x 64 bf16 tile.  Lane l loads chunk
// (l & 7) of rows (l >> 3) + 4 i, i < 4.
struct StepLoad {
  uint4 u[4];
};

// Stage the step into the warp's swizzled tile (chunk c of row kk at
// c ^ (kk & 7)) and accumulate coef(16 x 16) x tile into D.
template <bool kTwo = false>
__device__ __forceinline__ void mma_step(Frag& D, const StepLoad& s, uint32_t tile, const uint32_t (&a)[4],
                                         int lane, const uint32_t* a2 = nullptr) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int kk = (lane >> 3) + 4 * i, c = lane & 7;
    sts4(tile + static_cast<uint32_t>(kk * 8 + (c ^ (kk & 7))) * 16u, s.u[i]);
  }
  __syncwarp();
#pragma unroll
  for (int p = 0; p < 4; ++p) {  // n-blocks 2p, 2p + 1
    const int kk = (lane & 7) + 8 * ((lane >> 3) & 1), cc = 2 * p + (lane >> 4);
    uint32_t r0, r1, r2, r3;
    ldsm_x4_trans(tile + static_cast<uint32_t>(kk * 8 + (cc ^ (kk & 7))) * 16u, r0, r1, r2, r3);
    mma_bf16(D.d[2 * p], a, r0, r1);
    mma_bf16(D.d[2 * p + 1], a, r2, r3);
    if constexpr (kTwo) {  // a second coefficient set on the same staged rows
      const uint32_t b4[4] = {a2[0], a2[1], a2[2], a2[3]};
      mma_bf16(D.d[2 * p], b4, r0, r1);
      mma_bf16(D.d[2 * p + 1], b4, r2, r3);
    }
  }
  __syncwarp();  // the tile is rewritten by the next step
}

// ---- tcgen05 (5th-generation tensor cores, accumulators in TMEM) ----
// Shared-memory matrix descriptor, no swizzle ("interleave"): core matrices
// of 8 rows x 16 bytes, LBO / SBO the byte strides between core matrices
// along the leading (K) / strided dimension (cute UMMA::SmemDescriptor,
// version 1 for sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3fffu) | (static_cast<uint64_t>((lbo >> 4) & 0x3fffu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}
// kind::f16 instruction descriptor: D f32, A and B bf16, A MN-major, B K-major, M = 128, N = 16.
constexpr uint32_t kIdescM128N16 = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((16u >> 3) << 17) |
                                   ((128u >> 4) << 24);

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdescM128N16), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Products of one cooperative ring stage (16 rows x 1 KB, 16-byte chunk c of
// row kk at (c & ~7) | ((c ^ kk) & 7)): warp cw takes chunks 8 cw .. 8 cw + 7.
template <bool kTwo>
__device__ __forceinline__ void mma_ring(Frag& D, uint32_t stage, const uint32_t (&a)[4], const uint32_t* a2, int cw,
                                         int lane) {
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int kk = (lane & 7) + 8 * ((lane >> 3) & 1), cc = 8 * cw + 2 * p + (lane >> 4);
    const int pos = (cc & ~7) | ((cc ^ kk) & 7);
    uint32_t r0, r1, r2, r3;
    ldsm_x4_trans(stage + static_cast<uint32_t>(kk * 64 + pos) * 16u, r0, r1, r2, r3);
    mma_bf16(D.d[2 * p], a, r0, r1);
    mma_bf16(D.d[2 * p + 1], a, r2, r3);
    if constexpr (kTwo) {
      const uint32_t b4[4] = {a2[0], a2[1], a2[2], a2[3]};
      mma_bf16(D.d[2 * p], b4, r0, r1);
      mma_bf16(D.d[2 * p + 1], b4, r2, r3);
    }
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// The batched forward of one linear.
// ---------------------------------------------------------------------------
struct BatchSmem {
  uint32_t cuts, xs, xu, lw, lu, msk, misc, tiles, ring, btile, mbar, tco, red, total;
  __host__ __device__ static uint32_t up(uint32_t v) { return (v + 15u) / 16u * 16u; }
  __host__ __device__ static BatchSmem make(const BatchParams& P) {
    BatchSmem L;
    uint32_t o = 0;
    L.cuts = o;
    o += 8u * kBatchMax;
    L.misc = o;
    o += 4u * 96;
    L.xs = o;  // [B][range] bf16
    o = up(o + 2u * P.B * P.range_max);
    L.xu = o;  // [B][slice] bf16
    o = up(o + 2u * P.B * P.slice_max);
    L.lw = o;  // {channel, token mask} of U in the W range
    o = up(o + 8u * P.range_max);
    L.lu = o;  // {channel, token mask} of the complements in the stage-1 slice
    o = up(o + 8u * P.slice_max);
    L.msk = o;  // token masks of one range (list building scratch)
    o = up(o + 4u * static_cast<uint32_t>((P.range_max > P.slice_max ? P.range_max : P.slice_max) + 64));
    L.tiles = o;  // per warp: one 16 x 64 bf16 step tile
    o += static_cast<uint32_t>(kWarps) * kStage * 128u;
    L.ring = o;  // cw == 8: CTA-cooperative ring of kRing 16-row x 1 KB stages
    const uint32_t nring = P.cw == 8 ? static_cast<uint32_t>(P.tc ? kRingT : kRing) : 0u;
    o += nring * kStage * 1024u;
    L.btile = o;  // tcgen05: per ring slot, the B operands (coefficients, hi and lo) 2 x 512 B
    o += P.tc ? nring * 1024u : 0u;
    L.mbar = o;   // tcgen05: per ring slot, the MMA-completion mbarrier; then the TMEM address
    o += 8u * kRingT + 16u;
    L.tco = o;  // t of the CTA's A rows: [hi/lo][B][na] bf16
    o = up(o + 4u * P.B * P.na_max);
    L.red = o;  // cross-group reduction [RG][16][64 CW] fp32
    o += 4u * 16u * static_cast<uint32_t>(kWarps) * kColsPerWarp;
    L.total = o;  // (CTAs b < B also run a cut from L.lw on: batch_smem_bytes)
    return L;
  }
};

__device__ long long g_batch_trace[160 * 16];

__global__ void __launch_bounds__(kThreads, 1) batch_forward_kernel(const BatchParams P) {
  extern __shared__ __align__(16) uint8_t smem_bf[];
  long long t_start;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_start));
#define BT_STAMP(i)                                                        \
  do {                                                                     \
    if (P.trace && threadIdx.x == 0) {                                     \
      long long c_;                                                        \
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_));                  \
      g_batch_trace[blockIdx.x * 16 + (i)] = c_ - t_start;                 \
    }                                                                      \
  } while (0)
  const BatchSmem L = BatchSmem::make(P);
  const uint32_t sb = smem_base_pinned(smem_bf);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int bid = blockIdx.x, NB = gridDim.x, KS = P.ks, B = P.B;
  const int ct = bid / KS, ks = bid - ct * KS;
  const int CW = P.cw, RG = kWarps / CW, cw = warp % CW, rg = warp / CW;
  const int wc0 = bpart(P.n, ks, KS), wc1 = bpart(P.n, ks + 1, KS);
  const int uc0 = bpart(P.n, bid, NB), uc1 = bpart(P.n, bid + 1, NB);
  const bool has_lr = P.r > 0 && P.k < P.n;
  const int alo = has_lr ? bpart(P.r, ks, KS) : 0, ahi = has_lr ? bpart(P.r, ks + 1, KS) : 0, na = ahi - alo;
  const int colw = ct * kColsPerWarp * CW + cw * kColsPerWarp;  // this warp's first output column
  const uint32_t tile = sb + L.tiles + static_cast<uint32_t>(warp) * kStage * 128u;
  const uint64_t pol = l2_evict_first_policy();

  // ---- CTA b < B computes token b's exact cut (the batch-1 selector) in the
  // memory past the activation slabs, published to the grid through ctr[2] ----
  SelArea C;
  C.h1 = sb + L.lw;
  C.cand = C.h1 + 4u * kBins;
  C.h2a = C.cand + 4u * kCandWords;
  C.h2b = C.h2a + 4u * 256;
  C.misc = C.h2b + 4u * 256;
  C.h16 = C.misc + 4u * kMiscWords;
  C.xs = C.h16 + 4u * kH16Words;
  C.zero = P.zero;
  if (bid < B) sel_clear16(C);  // x-independent: overlaps the previous launch under PDL
  if (tid == 0 && has_lr && uc1 > uc0)  // the stage-1 slice of B_r^T (contiguous) towards L2 meanwhile
    prefetch_l2_bulk(static_cast<const uint8_t*>(P.Bt) + static_cast<size_t>(uc0) * P.r_pad * 2,
                     static_cast<uint32_t>(uc1 - uc0) * static_cast<uint32_t>(P.r_pad) * 2u);
  if (P.pdl) {
    griddep_wait();  // the previous launch's y (our x) and workspace are complete
    griddep_launch_dependents();
  }
  if (bid < B) {
    __syncthreads();  // the cleared histogram
    sel_load16(static_cast<const uint8_t*>(P.x) + static_cast<size_t>(bid) * P.n * 2, P.n, C);
    const Cut cut = sel_cut16(P.n, P.k, C);
    if (tid == 0) {
      P.cuts[bid] = make_int2(static_cast<int>(cut.T), cut.jlim);
      red_release_add(P.ctr + 2, 1u);
    }
  }
  BT_STAMP(0);

  SelArea S{};  // compact2 scratch (misc counters)
  S.misc = sb + L.misc;

  // ---- the activations of the CTA's channel ranges, then the cuts ----
  // Activations of the CTA's channel ranges, all tokens, in shared memory:
  // rows start at the 8-aligned channels wb0 / ub0 (16-byte vectors).
  const int wb0 = wc0 & ~7, ub0 = uc0 & ~7;
  const uint16_t* x16 = static_cast<const uint16_t*>(P.x);
  // both ranges in one round trip: vectors [0, nvw) of the W range, then [0, nvu) of the slice
  if ((P.n & 7) == 0) {
    const int nvw = (wc1 - wb0 + 7) >> 3, nvu = has_lr ? (uc1 - ub0 + 7) >> 3 : 0;
    for (int v = tid; v < nvw + nvu; v += kThreads) {
      const bool w_side = v < nvw;
      const int vv = w_side ? v : v - nvw;
      const int c0 = w_side ? wb0 : ub0;
      const uint32_t dst = (w_side ? sb + L.xs : sb + L.xu) + 16u * vv;
      const int stride = w_side ? P.range_max : P.slice_max;
      uint4 u[kBatchMax];
#pragma unroll
      for (int b = 0; b < kBatchMax; ++b)
        if (b < B) u[b] = __ldg(reinterpret_cast<const uint4*>(x16 + static_cast<size_t>(b) * P.n + c0) + vv);
#pragma unroll
      for (int b = 0; b < kBatchMax; ++b)
        if (b < B) sts4(dst + 2u * (b * stride), u[b]);
    }
  } else {
    for (int b = 0; b < B; ++b) {
      for (int jj = tid; jj < wc1 - wb0; jj += kThreads)
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(sb + L.xs + 2u * (b * P.range_max + jj)),
                     "h"(x16[static_cast<size_t>(b) * P.n + wb0 + jj]) : "memory");
      for (int jj = tid; has_lr && jj < uc1 - ub0; jj += kThreads)
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(sb + L.xu + 2u * (b * P.slice_max + jj)),
                     "h"(x16[static_cast<size_t>(b) * P.n + ub0 + jj]) : "memory");
    }
  }
  if (tid == 0) spin_until_count(P.ctr + 2, static_cast<unsigned>(B));
  __syncthreads();
  if (tid < B) {
    const int2 c = __ldcg(P.cuts + tid);
    sts2(sb + L.cuts + 8u * tid, static_cast<uint32_t>(c.x), static_cast<uint32_t>(c.y));
  }
  __syncthreads();
  BT_STAMP(1);
  // (after the cut: its scratch overlaps the ring, the mbarriers and the TMEM slot)
  const bool tc = P.tc && CW == 8;  // W and stage-2 products on tcgen05 (TMEM accumulators)
  uint32_t tmem = 0;
  if (tc) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(sb + L.mbar + 8u * kRingT)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
      for (int q = 0; q < kRingT; ++q) mbar_init_s(sb + L.mbar + 8u * q, 1);
      fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    tmem = lds(sb + L.mbar + 8u * kRingT);
  }
  const uint32_t all = (1u << B) - 1u;
  // Token masks of channels j2, j2 + 1 (j2 even): bit b = channel in S_b
  // (packed-pair key tests against each token's cut).
  auto token_masks2 = [&](uint32_t xr, int stride, int base, int j2, uint32_t& t0, uint32_t& t1) {
    t0 = t1 = 0u;
    for (int b = 0; b < B; ++b) {
      const uint2 c = lds2(sb + L.cuts + 8u * b);
      const uint32_t w = lds(xr + 2u * (b * stride + (j2 - base)));
      if (c.x <= 0x7fff0000u) {
        const uint32_t t15 = c.x >> 16;
        const uint32_t gt = t15 < 0x7fffu ? pair_gt(w, t15) : 0u;
        const uint32_t eq = pair_eq(w, t15);
        const int jl = static_cast<int>(c.y) - j2;  // channels below jlim: j2 if jl > 0, j2 + 1 if jl > 1
        t0 |= ((((gt >> 15) & 1u) | (((eq >> 15) & 1u) & static_cast<uint32_t>(jl > 0)))) << b;
        t1 |= ((((gt >> 31) & 1u) | (((eq >> 31) & 1u) & static_cast<uint32_t>(jl > 1)))) << b;
      }
    }
  };
  // Ascending list of {channel, token mask} over [lo, hi): the channels some
  // token selects (want_s) or some token leaves to the low-rank term
  // (!want_s).  64-channel chunks over all warps, ballot prefix sums.
  // Two __syncthreads.
  auto build_list = [&](uint32_t xr, int stride, int lo, int hi, bool want_s, uint32_t list, int slot) {
    const int base = lo & ~7;
    const int lo2 = lo & ~1;
    const int nch = hi > lo ? (hi - lo2 + 63) >> 6 : 0;
    const int per = (nch + kWarps - 1) / kWarps, ch0 = min(nch, warp * per), ch1 = min(nch, (warp + 1) * per);
    auto members = [&](int j2, uint32_t& t0, uint32_t& t1) {
      const int jr = min(j2, (hi - 1) & ~1);  // in-range load address
      token_masks2(xr, stride, base, jr, t0, t1);
      if (!want_s) {
        t0 = all & ~t0;
        t1 = all & ~t1;
      }
      const uint32_t m = static_cast<uint32_t>(t0 != 0u) | (static_cast<uint32_t>(t1 != 0u) << 1);
      const int lo_off = min(max(lo - j2, 0), 2), hi_off = min(max(hi - j2, 0), 2);
      return m & ((1u << hi_off) - 1u) & ~((1u << lo_off) - 1u);
    };
    uint32_t cnt = 0;
    for (int c = ch0; c < ch1; ++c) {  // pass 1: masks -> scratch, counts
      uint32_t t0, t1;
      const int j2 = lo2 + 64 * c + 2 * lane;
      const uint32_t m = members(j2, t0, t1);
      cnt += __popc(m);
      sts2(sb + L.msk + 4u * static_cast<uint32_t>(j2 - lo2), t0 | (m << 30), t1);
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) S.set_m(slot + warp, cnt);
    __syncthreads();
    uint32_t off = 0, tot = 0;
#pragma unroll
    for (int q = 0; q < kWarps; ++q) {
      const uint32_t v = S.m(slot + q);
      off += q < warp ? v : 0u;
      tot += v;
    }
    const uint32_t lt = lanemask_lt();
    for (int c = ch0; c < ch1; ++c) {  // pass 2: from the scratch
      const int j2 = lo2 + 64 * c + 2 * lane;
      const uint2 tt = lds2(sb + L.msk + 4u * static_cast<uint32_t>(j2 - lo2));
      const uint32_t m = tt.x >> 30, t0 = tt.x & 0x3fffffffu, t1 = tt.y;
      const uint32_t bal0 = __ballot_sync(0xffffffffu, m & 1u), bal1 = __ballot_sync(0xffffffffu, (m >> 1) & 1u);
      const uint32_t pre = off + __popc(bal0 & lt) + __popc(bal1 & lt);
      sts2_pred(m & 1u, list + 8u * pre, static_cast<uint32_t>(j2), t0);
      sts2_pred((m >> 1) & 1u, list + 8u * (pre + (m & 1u)), static_cast<uint32_t>(j2 + 1), t1);
      off += __popc(bal0) + __popc(bal1);
    }
    __syncthreads();
    return static_cast<int>(tot);
  };
  const int nW = build_list(sb + L.xs, P.range_max, wc0, wc1, true, sb + L.lw, M_LISTA);
  const int nU = has_lr ? build_list(sb + L.xu, P.slice_max, uc0, uc1, false, sb + L.lu, M_LISTB) : 0;
  BT_STAMP(2);

  // A fragment of gathered rows: coef(m, kk) = mask_m ? x_m[row kk] : 0,
  // rows from list entries e0 + stride * kk (kk < 16, beyond cnt: 0).
  auto frag_list = [&](uint32_t list, int e0, int stride, int cnt, uint32_t xr, int xstride, int jbase,
                       uint32_t (&a)[4]) {
    uint32_t lo[2][2], hi[2][2];  // [row pair 2t / 2t+8][token g / g+8] as (k, k+1) halves
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int kk = 2 * t4 + 8 * h + q;
        const int e = e0 + stride * kk;
        const bool ok = e < cnt;
        const uint2 ent = lds2(list + 8u * static_cast<uint32_t>(ok ? e : 0));
        const int jj = static_cast<int>(ent.x) - jbase;
        // unconditional loads (clamped token rows), masked values: no branches
        const uint32_t m0 = ok ? (ent.y >> g) & 1u : 0u, m1 = ok ? (ent.y >> (g + 8)) & 1u : 0u;
        const uint32_t v0 = lds_u16(xr + 2u * (min(g, B - 1) * xstride + jj)) & (0u - m0);
        const uint32_t v1 = lds_u16(xr + 2u * (min(g + 8, B - 1) * xstride + jj)) & (0u - m1);
        if (q == 0) {
          lo[h][0] = v0;
          lo[h][1] = v1;
        } else {
          hi[h][0] = v0;
          hi[h][1] = v1;
        }
      }
    }
    a[0] = pack_bf16(lo[0][0], hi[0][0]);
    a[1] = pack_bf16(lo[0][1], hi[0][1]);
    a[2] = pack_bf16(lo[1][0], hi[1][0]);
    a[3] = pack_bf16(lo[1][1], hi[1][1]);
  };
  // Loads of one step: rows from `rowaddr(kk)` (16-B aligned segment start),
  // chunks >= vch clamped to chunk 0 (their columns are discarded).
  auto load_step = [&](StepLoad& s, auto&& rowaddr, int vch) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int kk = (lane >> 3) + 4 * i, c = lane & 7;
      s.u[i] = ldg_stream_ef(static_cast<const uint8_t*>(rowaddr(kk)) + 16 * (c < vch ? c : 0), pol);
    }
  };
  auto zero_frag = [&](Frag& D) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int e = 0; e < 4; ++e) D.d[q][e] = 0.f;
  };
  // Run `nsteps` steps with kDepth in flight: rows(step, kk) -> address,
  // coef(step, a, a2) -> one (or, kTwo, two) coefficient fragments,
  // done(step) after each step's products.
  auto run_steps = [&](auto two, Frag& D, int nsteps, auto&& rowaddr_of, auto&& coef_of, auto&& vch_of,
                       auto&& done) {
    constexpr bool kTwo = decltype(two)::value;
    StepLoad s[kDepth];
#pragma unroll
    for (int d = 0; d < kDepth; ++d)
      if (d < nsteps) load_step(s[d], [&](int kk) { return rowaddr_of(d, kk); }, vch_of(d));
    for (int st0 = 0; st0 < nsteps; st0 += kDepth) {
#pragma unroll
      for (int d = 0; d < kDepth; ++d) {
        const int st = st0 + d;
        if (st < nsteps) {
          uint32_t a[4], a2[4];
          coef_of(st, a, a2);
          mma_step<kTwo>(D, s[d], tile, a, lane, a2);
          done(st);
          if (st + kDepth < nsteps)
            load_step(s[d], [&](int kk) { return rowaddr_of(st + kDepth, kk); }, vch_of(st + kDepth));
        }
      }
    }
  };
  auto nothing = [](int) {};
  // cw == 8: all warps share each step's 16 rows x 1 KB (the CTA's whole
  // column tile), staged by cp.async in a kRing-deep ring -- every row tile is
  // fetched as one contiguous 1 KB run by the CTA at once.
  auto coop_steps = [&](auto two, Frag& D, int nsteps, auto&& rowseg, int vbytes, auto&& coef_of) {
    constexpr bool kTwo = decltype(two)::value;
    auto issue = [&](int st) {
      if (st < nsteps) {
        const uint32_t stage = sb + L.ring + static_cast<uint32_t>(st % kRing) * kStage * 1024u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int id = tid + kThreads * q, kk = id >> 6, c = id & 63;
          const uint8_t* src = static_cast<const uint8_t*>(rowseg(st, kk)) + 16 * (c * 16 < vbytes ? c : 0);
          cp_async16_s_ef(stage + static_cast<uint32_t>(kk * 64 + ((c & ~7) | ((c ^ kk) & 7))) * 16u, src, pol);
        }
      }
      cp_async_commit();
    };
#pragma unroll
    for (int q = 0; q < kRing - 1; ++q) issue(q);
    for (int st = 0; st < nsteps; ++st) {
      cp_async_wait_group<kRing - 2>();
      __syncthreads();
      uint32_t a[4], a2[4];
      coef_of(st, a, a2);
      mma_ring<kTwo>(D, sb + L.ring + static_cast<uint32_t>(st % kRing) * kStage * 1024u, a, a2, cw, lane);
      __syncthreads();  // the stage is refilled below
      issue(st + kRing - 1);
    }
    cp_async_wait_group<0>();
  };

  // tcgen05 version of coop_steps: the ring stage in the MN-major interleave
  // layout (chunk c of row kk: core matrix (c, kk / 8) at (2 c + kk / 8) x 128 B),
  // the step's coefficients as a K-major 16 x 16 B operand, one thread issuing
  // four M = 128 MMAs per step into the TMEM accumulator (column block q of the
  // 512-column tile at TMEM columns 16 q), a commit per step to the slot's
  // mbarrier (the slot is refilled once its MMAs have read it).
  int gstep = 0;            // ring steps issued so far (slot = gstep % kRingT, parity = gstep / kRingT)
  uint32_t tc_acc = 0;      // the accumulator holds data
  auto tc_steps = [&](auto two, int nsteps, auto&& rowseg, int vbytes, auto&& coefB) {
    constexpr bool kTwo = decltype(two)::value;
    const int g0 = gstep;
    auto issue = [&](int st) {
      if (st < nsteps) {
        const uint32_t stage = sb + L.ring + static_cast<uint32_t>((g0 + st) % kRingT) * kStage * 1024u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int id = tid + kThreads * q, kk = id >> 6, c = id & 63;
          const uint8_t* src = static_cast<const uint8_t*>(rowseg(st, kk)) + 16 * (c * 16 < vbytes ? c : 0);
          cp_async16_s_ef(stage + static_cast<uint32_t>((2 * c + (kk >> 3)) * 128 + (kk & 7) * 16), src, pol);
        }
      }
      cp_async_commit();
    };
    auto wait_slot = [&](int gs) {  // MMAs of global step gs have completed
      mbar_wait_s(sb + L.mbar + 8u * static_cast<uint32_t>(gs % kRingT), static_cast<uint32_t>((gs / kRingT) & 1));
    };
    constexpr int kLook = kRingT - 2;  // steps in flight ahead of the MMAs
#pragma unroll
    for (int q = 0; q < kLook; ++q) issue(q);
    for (int st = 0; st < nsteps; ++st) {
      const int gs = g0 + st, slot = gs % kRingT;
      cp_async_wait_group<kLook - 1>();
      // coefficients (B operand, K-major interleave: (n, k) at ((n/8) 2 + k/8) 128 + (n%8) 16 + (k%8) 2)
      const uint32_t bt = sb + L.btile + static_cast<uint32_t>(slot) * 1024u;
      {
        const int n = tid >> 4, k = tid & 15;
        const uint32_t off = static_cast<uint32_t>(((n >> 3) * 2 + (k >> 3)) * 128 + (n & 7) * 16 + (k & 7) * 2);
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(bt + off), "h"(static_cast<unsigned short>(coefB(st, 0, n, k)))
                     : "memory");
        if constexpr (kTwo)
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(bt + 512u + off),
                       "h"(static_cast<unsigned short>(coefB(st, 1, n, k)))
                       : "memory");
      }
      fence_proxy_async_smem();  // this thread's cp.async data and coefficients -> the async proxy
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        const uint32_t stage = sb + L.ring + static_cast<uint32_t>(slot) * kStage * 1024u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint64_t ad = umma_desc(stage + 4096u * q, 128u, 256u);
          tc_mma(tmem + 16u * q, ad, umma_desc(bt, 128u, 256u), tc_acc);
          if constexpr (kTwo) tc_mma(tmem + 16u * q, ad, umma_desc(bt + 512u, 128u, 256u), 1u);
        }
        tc_commit(sb + L.mbar + 8u * static_cast<uint32_t>(slot));
      }
      tc_acc = 1u;
      // refill the slot of step gs - 2 once its MMAs are done (long since, normally)
      if (st >= 2) wait_slot(gs - 2);
      issue(st + kLook);
    }
    if (nsteps > 1) wait_slot(g0 + nsteps - 2);
    if (nsteps > 0) wait_slot(g0 + nsteps - 1);
    cp_async_wait_group<0>();
    gstep = g0 + nsteps;
  };

  const __nv_bfloat16* Wt = static_cast<const __nv_bfloat16*>(P.Wt);
  const __nv_bfloat16* At = static_cast<const __nv_bfloat16*>(P.At);
  const __nv_bfloat16* Bt = static_cast<const __nv_bfloat16*>(P.Bt);

  // ---- stage 1: t_b += sum over the slice's complement rows (all r columns).
  // Warp w owns 64-column chunks w, w + 8, ...; its steps run chunk after
  // chunk in one pipeline (the next chunk's rows load while the previous
  // chunk finishes), and each chunk is reduced into the L2 t accumulator once. ----
  if (has_lr && nU > 0) {
    const int nch = (P.r_pad + kColsPerWarp - 1) / kColsPerWarp;
    const int nsteps = (nU + kStage - 1) / kStage;
    const int mych = nch > warp ? (nch - warp + kWarps - 1) / kWarps : 0;
    Frag Dt;
    zero_frag(Dt);
    run_steps(
        std::false_type{}, Dt, mych * nsteps,
        [&](int i, int kk) {
          const int qi = i / nsteps, st = i - qi * nsteps, q = warp + kWarps * qi;
          const int e = min(st * kStage + kk, nU - 1);
          const uint32_t j = lds(sb + L.lu + 8u * static_cast<uint32_t>(e));
          return static_cast<const void*>(Bt + static_cast<size_t>(j) * P.r_pad + q * kColsPerWarp);
        },
        [&](int i, uint32_t(&a)[4], uint32_t(&)[4]) {
          const int qi = i / nsteps, st = i - qi * nsteps;
          frag_list(sb + L.lu, st * kStage, 1, nU, sb + L.xu, P.slice_max, ub0, a);
        },
        [&](int i) {
          const int q = warp + kWarps * (i / nsteps);
          return min(8, (P.r_pad - q * kColsPerWarp) / 8);
        },
        [&](int i) {
          const int qi = i / nsteps, st = i - qi * nsteps;
          if (st != nsteps - 1) return;
          const int c0 = (warp + kWarps * qi) * kColsPerWarp;
#pragma unroll
          for (int nb = 0; nb < 8; ++nb) {
            const int c = c0 + 8 * nb + 2 * t4;
            if (c < P.r_pad) {
              if (g < B) red_add_v2(P.t_acc + static_cast<size_t>(g) * P.r_pad + c, Dt.d[nb][0], Dt.d[nb][1]);
              if (g + 8 < B) red_add_v2(P.t_acc + static_cast<size_t>(g + 8) * P.r_pad + c, Dt.d[nb][2], Dt.d[nb][3]);
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) Dt.d[nb][e] = 0.f;
          }
        });
  }
  if (P.zero_y) {  // this CTA's share of y, published by the arrival below (the combine waits for it)
    const int nv = B * P.m;
    const int v0 = bpart(nv, bid, NB), v1 = bpart(nv, bid + 1, NB);
    for (int i = v0 + tid; i < v1; i += kThreads) P.y[i] = 0.f;
  }
  __syncthreads();
  BT_STAMP(3);
  if (tid == 0) red_release_add(P.ctr, 1u);
  BT_STAMP(4);

  // ---- W rows of U (this warp: row group rg, columns [colw, colw + 64)) ----
  Frag D;
  zero_frag(D);
  {
    const int vch = max(0, min(8, (P.m_pad - colw) / 8));
    const int mine = nW > rg ? (nW - rg + RG - 1) / RG : 0;  // entries rg, rg + RG, ...
    const int nsteps = (mine + kStage - 1) / kStage;
    const int tcol0 = ct * kColsPerWarp * CW;
    if (tc)
      tc_steps(
          std::false_type{}, nsteps,
          [&](int st, int kk) {
            const int e = min(st * kStage + kk, nW - 1);
            const uint32_t j = lds(sb + L.lw + 8u * static_cast<uint32_t>(e));
            return static_cast<const void*>(Wt + static_cast<size_t>(j) * P.m_pad + tcol0);
          },
          min(1024, 2 * (P.m_pad - tcol0)),
          [&](int st, int, int n, int k) -> uint32_t {
            const int e = st * kStage + k;
            if (e >= nW || n >= B) return 0u;
            const uint2 ent = lds2(sb + L.lw + 8u * static_cast<uint32_t>(e));
            return ((ent.y >> n) & 1u) ? lds_u16(sb + L.xs + 2u * (n * P.range_max + (static_cast<int>(ent.x) - wb0)))
                                       : 0u;
          });
    else if (CW == 8)
      coop_steps(
          std::false_type{}, D, nsteps,
          [&](int st, int kk) {
            const int e = min(st * kStage + kk, nW - 1);
            const uint32_t j = lds(sb + L.lw + 8u * static_cast<uint32_t>(e));
            return static_cast<const void*>(Wt + static_cast<size_t>(j) * P.m_pad + tcol0);
          },
          min(1024, 2 * (P.m_pad - tcol0)),
          [&](int st, uint32_t(&a)[4], uint32_t(&)[4]) {
            frag_list(sb + L.lw, st * kStage, 1, nW, sb + L.xs, P.range_max, wb0, a);
          });
    else if (vch > 0)
      run_steps(
          std::false_type{}, D, nsteps,
          [&](int st, int kk) {
            const int e = rg + RG * min(st * kStage + kk, mine - 1);
            const uint32_t j = lds(sb + L.lw + 8u * static_cast<uint32_t>(e));
            return static_cast<const void*>(Wt + static_cast<size_t>(j) * P.m_pad + colw);
          },
          [&](int st, uint32_t(&a)[4], uint32_t(&)[4]) {
            frag_list(sb + L.lw, rg + RG * st * kStage, RG, nW, sb + L.xs, P.range_max, wb0, a);
          },
          [&](int) { return vch; }, nothing);
  }

  // ---- t barrier, then stage 2 over the A_r^T rows [alo, ahi) ----
  BT_STAMP(5);
  if (has_lr) {
    if (tid == 0) spin_until_count(P.ctr, static_cast<unsigned>(NB));
    __syncthreads();
    BT_STAMP(6);
    // t -> bf16 hi + lo (t ~= hi + lo to ~2^-16 relative), [hi/lo][b][c - alo]
    for (int i = tid; i < B * na; i += kThreads) {
      const int b = i / na, c = i - b * na;
      const float v = __ldcg(P.t_acc + static_cast<size_t>(b) * P.r_pad + alo + c);
      const __nv_bfloat16 h = __float2bfloat16_rn(v);
      const __nv_bfloat16 l = __float2bfloat16_rn(v - __bfloat162float(h));
      asm volatile("st.shared.u16 [%0], %1;" ::"r"(sb + L.tco + 2u * (b * P.na_max + c)),
                   "h"(__bfloat16_as_ushort(h)) : "memory");
      asm volatile("st.shared.u16 [%0], %1;" ::"r"(sb + L.tco + 2u * (B * P.na_max + b * P.na_max + c)),
                   "h"(__bfloat16_as_ushort(l)) : "memory");
    }
    __syncthreads();
    const int vch = max(0, min(8, (P.m_pad - colw) / 8));
    const int steps_all = (na + kStage - 1) / kStage;
    const int mine = steps_all > rg ? (steps_all - rg + RG - 1) / RG : 0;  // steps rg, rg + RG, ...
    const uint32_t th = sb + L.tco, tl = sb + L.tco + 2u * static_cast<uint32_t>(B * P.na_max);
    auto coef2 = [&](int cb, uint32_t(&a)[4], uint32_t(&a2)[4]) {
#pragma unroll
      for (int part_ = 0; part_ < 2; ++part_) {
        const uint32_t tc = part_ ? tl : th;
        uint32_t v[2][2][2];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int tk = 0; tk < 2; ++tk)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int c = cb + 2 * t4 + 8 * h + q, m = g + 8 * tk;
              v[h][tk][q] = lds_u16(tc + 2u * (min(m, B - 1) * P.na_max + min(c, na - 1))) &
                            (0u - static_cast<uint32_t>((c < na) & (m < B)));
            }
        uint32_t* o = part_ ? a2 : a;
        o[0] = pack_bf16(v[0][0][0], v[0][0][1]);
        o[1] = pack_bf16(v[0][1][0], v[0][1][1]);
        o[2] = pack_bf16(v[1][0][0], v[1][0][1]);
        o[3] = pack_bf16(v[1][1][0], v[1][1][1]);
      }
    };
    if (tc) {
      const int tcol0 = ct * kColsPerWarp * CW;
      tc_steps(
          std::true_type{}, steps_all,
          [&](int st, int kk) {
            const int c = min(st * kStage + kk, na - 1);
            return static_cast<const void*>(At + static_cast<size_t>(alo + c) * P.m_pad + tcol0);
          },
          min(1024, 2 * (P.m_pad - tcol0)),
          [&](int st, int part_, int n, int k) -> uint32_t {
            const int c = st * kStage + k;
            if (c >= na || n >= B) return 0u;
            return lds_u16((part_ ? tl : th) + 2u * (n * P.na_max + c));
          });
    } else if (CW == 8) {
      const int tcol0 = ct * kColsPerWarp * CW;
      coop_steps(
          std::true_type{}, D, steps_all,
          [&](int st, int kk) {
            const int c = min(st * kStage + kk, na - 1);
            return static_cast<const void*>(At + static_cast<size_t>(alo + c) * P.m_pad + tcol0);
          },
          min(1024, 2 * (P.m_pad - tcol0)), [&](int st, uint32_t(&a)[4], uint32_t(&a2)[4]) { coef2(st * kStage, a, a2); });
    } else if (vch > 0) {  // hi and lo coefficients on the same staged rows
      run_steps(
          std::true_type{}, D, mine,
          [&](int st, int kk) {
            const int c = min((rg + RG * st) * kStage + kk, na - 1);
            return static_cast<const void*>(At + static_cast<size_t>(alo + c) * P.m_pad + colw);
          },
          [&](int st, uint32_t(&a)[4], uint32_t(&a2)[4]) {
            const int cb = (rg + RG * st) * kStage;
#pragma unroll
            for (int part_ = 0; part_ < 2; ++part_) {
              const uint32_t tc = part_ ? tl : th;
              uint32_t v[2][2][2];
#pragma unroll
              for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int tk = 0; tk < 2; ++tk)
#pragma unroll
                  for (int q = 0; q < 2; ++q) {
                    const int c = cb + 2 * t4 + 8 * h + q, m = g + 8 * tk;
                    v[h][tk][q] = lds_u16(tc + 2u * (min(m, B - 1) * P.na_max + min(c, na - 1))) &
                                  (0u - static_cast<uint32_t>((c < na) & (m < B)));
                  }
              uint32_t* o = part_ ? a2 : a;
              o[0] = pack_bf16(v[0][0][0], v[0][0][1]);
              o[1] = pack_bf16(v[0][1][0], v[0][1][1]);
              o[2] = pack_bf16(v[1][0][0], v[1][0][1]);
              o[3] = pack_bf16(v[1][1][0], v[1][1][1]);
            }
          },
          [&](int) { return vch; }, nothing);
    }
  }

  BT_STAMP(7);
  // ---- combine the row groups, then y (split-K reductions at L2) ----
  const uint32_t red = sb + L.red;
  const int tcols = kColsPerWarp * CW;
  if (tc) {
    // TMEM lane m of column block q = output column 128 q + m, column n = token n
    if (warp < 4) {
      tc_fence_after();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t r[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(tmem + (static_cast<uint32_t>(32 * warp) << 16) + 16u * q));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int c = 128 * q + 32 * warp + lane;
#pragma unroll
        for (int n = 0; n < 16; ++n) sts(red + 4u * (n * tcols + c), tc_acc ? r[n] : 0u);
      }
    }
  } else {
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
      const int c = cw * kColsPerWarp + 8 * nb + 2 * t4;
      sts2(red + 4u * ((rg * 16 + g) * tcols + c), __float_as_uint(D.d[nb][0]), __float_as_uint(D.d[nb][1]));
      sts2(red + 4u * ((rg * 16 + g + 8) * tcols + c), __float_as_uint(D.d[nb][2]), __float_as_uint(D.d[nb][3]));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tc && warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
  const int col0 = ct * tcols;
  const bool vec = (P.m & 3) == 0;
  for (int i = tid; i < B * (tcols / 4); i += kThreads) {  // 4 consecutive columns per thread
    const int b = i / (tcols / 4), c = 4 * (i - b * (tcols / 4));
    if (col0 + c >= P.m) continue;
    float s4[4] = {0.f, 0.f, 0.f, 0.f};
    for (int q = 0; q < RG; ++q) {
      const uint4 u = lds4(red + 4u * ((q * 16 + b) * tcols + c));
      s4[0] += __uint_as_float(u.x);
      s4[1] += __uint_as_float(u.y);
      s4[2] += __uint_as_float(u.z);
      s4[3] += __uint_as_float(u.w);
    }
    float* yp = P.y + static_cast<size_t>(b) * P.m + col0 + c;
    if (vec && col0 + c + 3 < P.m) {
      if (KS > 1)
        red_add_v4(yp, s4[0], s4[1], s4[2], s4[3]);
      else
        *reinterpret_cast<float4*>(yp) = make_float4(s4[0], s4[1], s4[2], s4[3]);
    } else {
      for (int e = 0; e < 4 && col0 + c + e < P.m; ++e) {
        if (KS > 1)
          red_add_f32(yp + e, s4[e]);
        else
          yp[e] = s4[e];
      }
    }
  }

  // ---- the last CTA leaves the t accumulator and the counters zero ----
  __syncthreads();
  BT_STAMP(8);
  if (tid == 0) S.set_m(0, atom_add_acq_rel_gpu(P.ctr + 1, 1u) == static_cast<unsigned>(NB - 1));
  __syncthreads();
  if (S.m(0)) {
    for (int i = tid; i < B * P.r_pad; i += kThreads) P.t_acc[i] = 0.f;
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      P.ctr[0] = 0u;
      P.ctr[1] = 0u;
      P.ctr[2] = 0u;
    }
  }
}

size_t batch_smem_bytes(const BatchParams& p) {
  const BatchSmem L = BatchSmem::make(p);
  return std::max<size_t>(L.total, L.lw + select_smem_bytes(p.n, true));
}

cudaError_t batch_trace_copy(long long* host, int count) {
  return cudaMemcpyFromSymbol(host, g_batch_trace, sizeof(long long) * static_cast<size_t>(count) * 16);
}

cudaError_t launch_batch(const BatchParams& p, bool x_bf16, cudaStream_t stream) {
  if (!x_bf16) return cudaErrorInvalidValue;
  const size_t smem = batch_smem_bytes(p);
  cudaError_t e = cudaFuncSetAttribute(batch_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = p.pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, batch_forward_kernel, p);
}

}  // namespace rsp
