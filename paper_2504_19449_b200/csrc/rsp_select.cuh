// rsp_select.cuh -- exact block-wide top-k cut on |x| (one CTA of kThreads).
//
// Reference semantics (matrix.cpp:100-117, sparsity.cpp:20-32): S = the k
// channels of largest |x|, ties broken toward the LOWER index; S and its
// complement are reported in ascending index order.
//
// Keys are fp32 bit patterns with the sign cleared (bf16 activations are
// widened exactly: bits << 16).  For finite values their unsigned order is
// the order of fabs() on the values widened to double -- what the reference
// compares -- and +0/-0 share key 0 (a tie, broken by index).
//
// The result is a cut (T, jlim):   j in S  <=>  key_j > T  or  (key_j == T and j < jlim).
//
// Algorithm (x resident in shared memory, every thread sees the result):
//   level 1  4096-bin histogram of key bits 30..19 (exponent + 4 mantissa
//            bits) with plain shared atomics while x is loaded; per-warp bin
//            totals (redux) locate the warp, then the bin, holding the k-th
//            largest key;
//   gather   the bin's members (typically <1% of n) into an ascending list
//            (count, offsets, write over contiguous per-warp ranges -- no
//            shared counter: measured, a CTA-wide atomic counter costs ~3k
//            cycles and match.any ~300 cycles per call);
//   refine   block-parallel histograms of the members on the remaining key
//            bits: 18..16 for bf16 activations (then the key is exact),
//            18..11 / 10..3 / 2..0 for fp32, stopping when a sub-bin is taken whole;
//   ties     when the cut splits the channels of the exact key T, one block
//            scan over the ascending member list finds the `need` lowest
//            indices (the reference's lower-index tie break).
#pragma once

#include <limits.h>
#include <stdint.h>

#include "rsp_device.cuh"

#ifndef RSP_SEL_STAMP
#define RSP_SEL_STAMP(i)
#endif

namespace rsp {

constexpr int kBins = 4096;   // level-1 histogram: key bits 30..19 (exponent + 4 mantissa bits)
constexpr int kH16Words = 16384;  // 32768 bf16 keys x 16-bit counters (n <= 65535)
constexpr int kCandWords = 2048;  // gathered boundary-bin members (more: refine over all of x)
constexpr int kMiscWords = 224;

// misc[] word slots
enum : int {
  M_SCAN = 0,  // [0, 16): block-scan scratch
  M_BIN = 16, M_ABOVE = 17, M_CNT = 18, M_T = 19, M_JLIM = 20, M_GEN = 21, M_LAST = 22,
  M_RCNT = 64,   // [64, 80): per-warp gathered member counts
  M_WSUM = 80,   // [80, 88): per-warp level-1 bin totals (kWarps <= 8)
  M_MBAR = 88,   // [88, 90): the stack kernel's operand mbarrier (8-byte aligned)
  M_LISTA = 32,  // [32, 48): per-warp member counts, list A
  M_LISTB = 48,  // [48, 64): per-warp member counts, list B
  M_TCNT = 23,   // tie members appended so far (fast tie path)
  M_OVER = 24,   // bf16 keys >= kWinHi (sel_load16)
  M_PLAN = 96,    // [96, 120): the stack kernel's per-CTA plan, slot 0
  M_PLAN1 = 128,  // [128, 152): plan slot 1
  M_DESC0 = 160,  // [160, 184): staged linear descriptor, slot 0
  M_DESC1 = 184,  // [184, 208): slot 1
  M_PEER = 208,   // [208, 224): the stack kernel's y destinations of the current linear (8 pointers)
};

struct Cut {
  uint32_t T;
  int jlim;
};

__device__ __forceinline__ bool in_cut(uint32_t key, int j, const Cut& c) {
  return key > c.T || (key == c.T && j < c.jlim);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return v;
}

// Shared-window addresses of the selector's arrays.
struct SelArea {
  uint32_t xs;    // [n] raw activations (u16 bf16 bits or u32 fp32 bits)
  uint32_t h1;    // [kBins] level-1 histogram of key >> 19
  uint32_t h16;   // [kH16Words] bf16 activations: full 15-bit key histogram, 16-bit counters
  uint32_t cand;  // [kCandWords] boundary-bin member indices, ascending
  uint32_t h2a;   // [256] refinement histograms (zero between cuts)
  uint32_t h2b;   // [256]
  uint32_t misc;  // [kMiscWords]
  uint32_t zero;  // 0 at run time, opaque to the compiler (load-batching dependences)
  __device__ __forceinline__ uint32_t m(int slot) const { return lds(misc + 4u * slot); }
  __device__ __forceinline__ void set_m(int slot, uint32_t v) const { sts(misc + 4u * slot, v); }
};

// fp32 bit pattern (sign cleared) of activation j.
template <bool XBF>
__device__ __forceinline__ uint32_t sel_key(SelArea s, int j) {
  if constexpr (XBF)
    return (lds_u16(s.xs + 2u * static_cast<uint32_t>(j)) << 16) & 0x7fffffffu;
  else
    return lds(s.xs + 4u * static_cast<uint32_t>(j)) & 0x7fffffffu;
}
template <bool XBF>
__device__ __forceinline__ uint32_t sel_bits(SelArea s, int j) {
  if constexpr (XBF)
    return lds_u16(s.xs + 2u * static_cast<uint32_t>(j)) << 16;
  else
    return lds(s.xs + 4u * static_cast<uint32_t>(j));
}

__device__ __forceinline__ void hist_add(SelArea s, uint32_t bits) {
  reds_add(s.h1 + 4u * ((bits & 0x7fffffffu) >> 19), 1u);
}

// Zero the histograms (independent of x: may run before
// griddepcontrol.wait).  Callers __syncthreads before sel_load.
__device__ __forceinline__ void sel_clear(SelArea s) {
  for (int i = threadIdx.x; i < kBins / 4; i += kThreads) sts4(s.h1 + 16u * i, make_uint4(0, 0, 0, 0));
  if (threadIdx.x < 64) sts4(s.h2a + 16u * threadIdx.x, make_uint4(0, 0, 0, 0));
  else if (threadIdx.x < 128) sts4(s.h2b + 16u * (threadIdx.x - 64), make_uint4(0, 0, 0, 0));
}

// x (global; bf16 or fp32, any alignment) -> s.xs, and (when `hist`) the
// level-1 histogram (s.h1 zeroed and published).  All of a thread's 16-byte
// loads of one round are issued before any is consumed.  Ends with __syncthreads.
// x is read at L2 (ld.global.cg), not through the read-only non-coherent
// path: inside a stack launch it may have been written by other CTAs (an
// earlier linear's output, another rank's rows), ordered by the dependency
// acquire.
template <bool XBF>
__device__ __forceinline__ void sel_load(const void* __restrict__ x, int n, SelArea s, bool hist) {
  constexpr int kPer = XBF ? 8 : 4;  // elements per 16 B
  const uintptr_t a = reinterpret_cast<uintptr_t>(x);
  if ((a & 15u) == 0 && (n % kPer) == 0) {
    const uint4* xv = reinterpret_cast<const uint4*>(x);
    const int nv = n / kPer;
    for (int base = 0; base < nv; base += 4 * kThreads) {
      uint4 u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = base + q * kThreads + static_cast<int>(threadIdx.x);
        u[q] = i < nv ? __ldcg(xv + i) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = base + q * kThreads + static_cast<int>(threadIdx.x);
        if (i >= nv) continue;
        sts4(s.xs + 16u * static_cast<uint32_t>(i), u[q]);
        if (hist) {
          const uint32_t w[4] = {u[q].x, u[q].y, u[q].z, u[q].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if constexpr (XBF) {
              hist_add(s, w[e] << 16);
              hist_add(s, w[e] & 0xffff0000u);
            } else {
              hist_add(s, w[e]);
            }
          }
        }
      }
    }
  } else {
    for (int j = threadIdx.x; j < n; j += kThreads) {
      uint32_t bits;
      if constexpr (XBF) {
        const uint16_t raw = static_cast<const uint16_t*>(x)[j];
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(s.xs + 2u * j), "h"(raw) : "memory");
        bits = static_cast<uint32_t>(raw) << 16;
      } else {
        bits = __ldcg(static_cast<const uint32_t*>(x) + j);
        sts(s.xs + 4u * j, bits);
      }
      if (hist) hist_add(s, bits);
    }
  }
  __syncthreads();
}

// One warp: descending search of an nb-bin histogram (nb in {8, 256}) for
// the need-th largest; lane 0 writes misc[M_BIN / M_ABOVE / M_CNT].
__device__ __forceinline__ void warp_find_desc(SelArea s, uint32_t hist, int nb, uint32_t need) {
  const int lane = threadIdx.x & 31;
  const int per = (nb + 31) >> 5;  // 1 or 8
  uint32_t c[8];
  uint32_t local = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int pos = lane * per + q;
    c[q] = (q < per && pos < nb) ? lds(hist + 4u * static_cast<uint32_t>(nb - 1 - pos)) : 0u;
    local += c[q];
  }
  uint32_t inc = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  uint32_t acc = inc - local;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (q < per && acc < need && need <= acc + c[q]) {
      s.set_m(M_BIN, static_cast<uint32_t>(nb - 1 - (lane * per + q)));
      s.set_m(M_ABOVE, acc);
      s.set_m(M_CNT, c[q]);
    }
    acc += c[q];
  }
}

// bf16 activations, n % 8 == 0: the 3 key bits left below the level-1 bin
// (bits 18..16) and the tie break.  Members of the bin are rare (<~1% of n),
// so a vectorized pass adds only members into an 8-bin histogram, one warp
// picks the sub-bin, and -- only when the cut splits the channels of the
// exact key T -- one more pass counts T's channels per thread (contiguous
// index runs) and a block scan finds the need-th lowest index.
// Serial work is done by one warp (all 16 warps issuing it would cost 4x:
// four warps share each scheduler).
static __device__ __noinline__ Cut sel_cut_bf16_tail(int n, SelArea s, uint32_t bin, uint32_t need) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nv = n >> 3;
  const int v0 = static_cast<int>(static_cast<uint32_t>(nv) * tid / kThreads);
  const int v1 = static_cast<int>(static_cast<uint32_t>(nv) * (tid + 1) / kThreads);
  const uint32_t bpat = bin << 3;  // (key16 & 0x7ff8) of the bin's members
  for (int v = v0; v < v1; ++v) {
    const uint4 u = lds4(s.xs + 16u * static_cast<uint32_t>(v));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t k16 = (w[e >> 1] >> (16 * (e & 1))) & 0x7fffu;
      if ((k16 & 0x7ff8u) == bpat) reds_add(s.h2a + 4u * (k16 & 7u), 1u);
    }
  }
  __syncthreads();
  RSP_SEL_STAMP(1);
  if (warp == 0) {
    // sub-bins 7..0 (descending) in lanes 0..7
    const uint32_t c = lane < 8 ? lds(s.h2a + 4u * (7 - lane)) : 0u;
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t hit = __ballot_sync(0xffffffffu, lane < 8 && inc - c < need && need <= inc);
    const int src = __ffs(hit) - 1;
    const uint32_t need2 = need - __shfl_sync(0xffffffffu, inc - c, src);
    const uint32_t cnt2 = __shfl_sync(0xffffffffu, c, src);
    const uint32_t T = (bin << 19) | (static_cast<uint32_t>(7 - src) << 16);
    if (lane < 8) sts(s.h2a + 4u * lane, 0u);  // leave the histogram zero for the next cut
    if (lane == 0) {
      s.set_m(M_T, need2 == cnt2 ? T - 1u : T);  // whole sub-bin in S: key >= T
      s.set_m(M_JLIM, 0u);
      s.set_m(M_BIN, need2 == cnt2 ? 0u : need2);  // ties to take (0: none)
    }
  }
  __syncthreads();
  RSP_SEL_STAMP(2);
  const uint32_t T = s.m(M_T), need2 = s.m(M_BIN);
  if (need2 == 0) return Cut{T, 0};
  const uint32_t t16 = T >> 16;
  uint32_t mine = 0;
  for (int v = v0; v < v1; ++v) {
    const uint4 u = lds4(s.xs + 16u * static_cast<uint32_t>(v));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) mine += ((w[e >> 1] >> (16 * (e & 1))) & 0x7fffu) == t16;
  }
  const uint32_t ex = block_excl_scan(mine, s.misc + 4u * M_SCAN, nullptr);
  if (ex < need2 && need2 <= ex + mine) {
    uint32_t c = ex;
    for (int v = v0; v < v1; ++v) {
      const uint4 u = lds4(s.xs + 16u * static_cast<uint32_t>(v));
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
      bool done = false;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (!done && ((w[e >> 1] >> (16 * (e & 1))) & 0x7fffu) == t16 && ++c == need2) {
          s.set_m(M_JLIM, static_cast<uint32_t>(8 * v + e + 1));
          done = true;
        }
      }
      if (done) break;
    }
  }
  __syncthreads();
  RSP_SEL_STAMP(3);
  return Cut{T, static_cast<int>(s.m(M_JLIM))};
}

// The exact cut for keeping k of the n activations in s.xs (level-1
// histogram in s.h1 complete, s.h2 zero).  Every thread returns the same Cut.
// Contains __syncthreads; latency-bound, so loads are batched ahead of their
// uses and every phase is block-parallel.
template <bool XBF>
static __device__ __noinline__ Cut sel_cut(int n, int k, SelArea s) {
  if (k <= 0) return Cut{0xffffffffu, 0};
  if (k >= n) return Cut{0u, INT_MAX};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t kk = static_cast<uint32_t>(k);
  // ---- level-1 boundary bin.  Thread t owns kPB bins, descending from the
  // top: bins [kBins - kPB (t+1), kBins - kPB t).  Per-warp totals (redux)
  // locate the warp, then the owning warp scans its lanes.
  {
    constexpr int kPB = kBins / kThreads;
    const uint32_t h = s.h1 + 4u * static_cast<uint32_t>(kBins - kPB * (tid + 1));
    uint32_t c[kPB];
#pragma unroll
    for (int q4 = 0; q4 < kPB / 4; ++q4) {
      const uint4 u = lds4(h + 16u * (kPB / 4 - 1 - q4));
      c[4 * q4 + 0] = u.w;
      c[4 * q4 + 1] = u.z;
      c[4 * q4 + 2] = u.y;
      c[4 * q4 + 3] = u.x;
    }
    uint32_t local = 0;
#pragma unroll
    for (int q = 0; q < kPB; ++q) local += c[q];
    const uint32_t wsum = __reduce_add_sync(0xffffffffu, local);
    if (lane == 0) s.set_m(M_WSUM + warp, wsum);
    __syncthreads();
    const uint32_t tw = lane < kWarps ? s.m(M_WSUM + lane) : 0u;
    uint32_t inc = tw;
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t owner = __ballot_sync(0xffffffffu, lane < kWarps && inc - tw < kk && kk <= inc);
    const int wb = __ffs(owner) - 1;
    if (warp == wb) {
      const uint32_t wabove = __shfl_sync(0xffffffffu, inc - tw, wb);
      uint32_t li = local;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, li, o);
        if (lane >= o) li += t;
      }
      uint32_t acc = wabove + li - local;
      if (acc < kk && kk <= acc + local) {
#pragma unroll
        for (int q = 0; q < kPB; ++q) {
          if (acc < kk && kk <= acc + c[q]) {
            s.set_m(M_BIN, static_cast<uint32_t>(kBins - 1 - kPB * tid - q));
            s.set_m(M_ABOVE, acc);
            s.set_m(M_CNT, c[q]);
          }
          acc += c[q];
        }
      }
    }
    __syncthreads();
  }
  RSP_SEL_STAMP(0);
  const uint32_t bin = s.m(M_BIN);
  uint32_t need = kk - s.m(M_ABOVE), cnt = s.m(M_CNT);
  if (cnt == need) return Cut{(bin << 19) - 1u, 0};  // the whole bin is in S (bin >= 1 since k < n)
  if constexpr (XBF) {
    if ((n & 7) == 0) return sel_cut_bf16_tail(n, s, bin, need);
  }
  // ---- gather the bin's members into an ascending flat list (two passes
  // over contiguous per-warp index ranges: count, offsets, write)
  const bool gathered = cnt <= static_cast<uint32_t>(kCandWords);
  __syncwarp();
  if (gathered) {
    const int r0 = static_cast<int>(static_cast<uint32_t>(n) * warp / kWarps);
    const int r1 = static_cast<int>(static_cast<uint32_t>(n) * (warp + 1) / kWarps);
    uint32_t mine = 0;
    for (int j0 = r0; j0 < r1; j0 += 128) {
      uint32_t kq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) kq[q] = j0 + 32 * q + lane < r1 ? sel_key<XBF>(s, j0 + 32 * q + lane) : 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        mine += __popc(__ballot_sync(0xffffffffu, j0 + 32 * q + lane < r1 && (kq[q] >> 19) == bin));
    }
    RSP_SEL_STAMP(4);
    if (lane == 0) s.set_m(M_RCNT + warp, mine);
    __syncthreads();
    RSP_SEL_STAMP(5);
    const uint32_t wc = lane < kWarps ? s.m(M_RCNT + lane) : 0u;
    uint32_t inc = wc;
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    uint32_t off = __shfl_sync(0xffffffffu, inc - wc, warp);
    const uint32_t lt = lanemask_lt();
    for (int j0 = r0; j0 < r1; j0 += 128) {
      uint32_t kq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) kq[q] = j0 + 32 * q + lane < r1 ? sel_key<XBF>(s, j0 + 32 * q + lane) : 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = j0 + 32 * q + lane;
        const bool mem = j < r1 && (kq[q] >> 19) == bin;
        const uint32_t bal = __ballot_sync(0xffffffffu, mem);
        if (mem) sts(s.cand + 4u * (off + __popc(bal & lt)), static_cast<uint32_t>(j));
        off += __popc(bal);
      }
    }
    RSP_SEL_STAMP(6);
    __syncthreads();
  }
  RSP_SEL_STAMP(1);
  // ---- refine on the remaining key bits: bf16 keys 18..16 (then exact),
  // fp32 keys 18..11, 10..3, 2..0.  Block-parallel histogram of the members.
  const int src_n = gathered ? static_cast<int>(cnt) : n;
  uint32_t prefix = bin << 19, pmask = 0x7ff80000u;
  constexpr int kLev = XBF ? 1 : 3;
#pragma unroll 1
  for (int lev = 0; lev < kLev; ++lev) {
    const int shift = XBF ? 16 : (lev == 0 ? 11 : lev == 1 ? 3 : 0);
    const int nb = (XBF || lev == 2) ? 8 : 256;
    const uint32_t dmask = static_cast<uint32_t>(nb - 1);
    const uint32_t hcur = (lev & 1) ? s.h2b : s.h2a;
    const uint32_t hnxt = (lev & 1) ? s.h2a : s.h2b;
    for (int i = tid; i < src_n; i += kThreads) {
      const int j = gathered ? static_cast<int>(lds(s.cand + 4u * i)) : i;
      const uint32_t key = sel_key<XBF>(s, j);
      if ((key & pmask) == prefix) reds_add(hcur + 4u * ((key >> shift) & dmask), 1u);
    }
    __syncthreads();
    if (warp == 0) warp_find_desc(s, hcur, nb, need);
    else if (tid - 32 < 256) sts(hnxt + 4u * (tid - 32), 0u);
    __syncthreads();
    need -= s.m(M_ABOVE);
    prefix |= s.m(M_BIN) << shift;
    pmask |= dmask << shift;
    cnt = s.m(M_CNT);
    if (tid < 256) sts(hcur + 4u * tid, 0u);  // leave both buffers zero for the next cut
    if (cnt == need) return Cut{prefix - 1u, 0};  // whole sub-bin in S
  }
  RSP_SEL_STAMP(2);
  // ---- ties: prefix is the exact k-th key T; the `need` lowest-index of its
  // `cnt` channels go to S.  Members are visited in ascending index order
  // (contiguous per-thread runs of the ascending member list).
  const uint32_t T = prefix;
  const int i0 = static_cast<int>(static_cast<uint32_t>(src_n) * tid / kThreads);
  const int i1 = static_cast<int>(static_cast<uint32_t>(src_n) * (tid + 1) / kThreads);
  uint32_t ties = 0;
  for (int i = i0; i < i1; ++i) {
    const int j = gathered ? static_cast<int>(lds(s.cand + 4u * i)) : i;
    ties += sel_key<XBF>(s, j) == T;
  }
  const uint32_t ex = block_excl_scan(ties, s.misc + 4u * M_SCAN, nullptr);
  if (ex < need && need <= ex + ties) {
    uint32_t c = ex;
    for (int i = i0; i < i1; ++i) {
      const int j = gathered ? static_cast<int>(lds(s.cand + 4u * i)) : i;
      if (sel_key<XBF>(s, j) == T && ++c == need) {
        s.set_m(M_JLIM, static_cast<uint32_t>(j + 1));
        break;
      }
    }
  }
  __syncthreads();
  RSP_SEL_STAMP(3);
  return Cut{T, static_cast<int>(s.m(M_JLIM))};
}

// ===========================================================================
// bf16 activations: |x| has 2^15 distinct keys, so ONE histogram of all of
// them (16-bit counters packed two per word, 64 KB, zeroed off the critical
// path) yields the exact k-th key with a single descending scan; only a tie
// at the cut needs one more pass (lowest `need` indices of the key).
// ===========================================================================
__device__ __forceinline__ void sel_clear16(SelArea s) {
  for (int i = threadIdx.x; i < kH16Words / 4; i += kThreads) sts4(s.h16 + 16u * i, make_uint4(0, 0, 0, 0));
  if (threadIdx.x < 64) sts4(s.h2a + 16u * threadIdx.x, make_uint4(0, 0, 0, 0));
  else if (threadIdx.x < 128) sts4(s.h2b + 16u * (threadIdx.x - 64), make_uint4(0, 0, 0, 0));
  if (threadIdx.x == 0) s.set_m(M_OVER, 0u);
}

__device__ __forceinline__ void hist16_add(SelArea s, uint32_t bf_bits /* bf16 << 16 */) {
  const uint32_t k15 = (bf_bits >> 16) & 0x7fffu;
  reds_add(s.h16 + 4u * (k15 >> 1), 1u << (16 * (k15 & 1u)));
}

// The histogram window scanned first: keys [kWinLo, kWinHi), |x| in
// [2^-40, 2^24) -- 8192 keys, 16 KB of the 64 KB histogram.  The exact cut
// falls there for any realistic activation vector; otherwise (counted: the
// keys at or above kWinHi, or too few keys in the window) the whole
// histogram is scanned.
constexpr uint32_t kWinHi = 151u << 7, kWinKeys = 8192u, kWinLo = kWinHi - kWinKeys;

// Packed-pair key tests on a word holding two bf16 activations (keys are
// the 15 magnitude bits of each half; every sum below stays inside its half).
//   bit 15 / 31 set  <=>  low / high key > t   (t < 0x7fff)
__device__ __forceinline__ uint32_t pair_gt(uint32_t w, uint32_t t) {
  return ((w & 0x7fff7fffu) + (0x7fffu - t) * 0x10001u) & 0x80008000u;
}
//   bit 15 / 31 set  <=>  low / high key == t   (t <= 0x7fff)
__device__ __forceinline__ uint32_t pair_eq(uint32_t w, uint32_t t) {
  const uint32_t z = (w & 0x7fff7fffu) ^ (t * 0x10001u);
  return ~(z + 0x7fff7fffu) & 0x80008000u;
}
// 8 channels' flags (bits 15 / 31 of four words, channel 2i / 2i+1 in word i) -> bits 0..7.
__device__ __forceinline__ uint32_t pack8(uint32_t f0, uint32_t f1, uint32_t f2, uint32_t f3) {
  const uint32_t t = (f0 >> 15) | (f1 >> 13) | (f2 >> 11) | (f3 >> 9);  // even at 0,2,4,6; odd at 16,18,20,22
  return (t & 0x55u) | ((t >> 15) & 0xaau);
}

// x (global, bf16) -> s.xs, the 15-bit histogram (s.h16 zero and published)
// and misc[M_OVER] = #keys >= kWinHi.  Ends with __syncthreads.
__device__ __forceinline__ void sel_load16(const void* __restrict__ x, int n, SelArea s) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(x);
  uint32_t over = 0;
  if ((a & 15u) == 0 && (n & 7) == 0) {
    const uint4* xv = reinterpret_cast<const uint4*>(x);
    const int nv = n >> 3;
    constexpr int kB = 8;  // n <= 16384 in one round trip
    for (int base = 0; base < nv; base += kB * kThreads) {
      uint4 u[kB];
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        const int i = base + q * kThreads + static_cast<int>(threadIdx.x);
        u[q] = i < nv ? __ldcg(xv + i) : make_uint4(0, 0, 0, 0);
      }
      // every histogram update waits on every load of the round (see stream_list)
      uint32_t dep = 0;
#pragma unroll
      for (int q = 0; q < kB; ++q) dep ^= u[q].x;
      dep &= s.zero;
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        const int i = base + q * kThreads + static_cast<int>(threadIdx.x);
        if (i >= nv) continue;
        sts4(s.xs + 16u * static_cast<uint32_t>(i), u[q]);
        const uint32_t w[4] = {u[q].x | dep, u[q].y, u[q].z, u[q].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          hist16_add(s, w[e] << 16);
          hist16_add(s, w[e] & 0xffff0000u);
        }
        over += __popc(pack8(pair_gt(w[0], kWinHi - 1), pair_gt(w[1], kWinHi - 1), pair_gt(w[2], kWinHi - 1),
                             pair_gt(w[3], kWinHi - 1)));
      }
    }
  } else {
    for (int j = threadIdx.x; j < n; j += kThreads) {
      const uint16_t raw = static_cast<const uint16_t*>(x)[j];
      asm volatile("st.shared.u16 [%0], %1;" ::"r"(s.xs + 2u * j), "h"(raw) : "memory");
      hist16_add(s, static_cast<uint32_t>(raw) << 16);
      over += (raw & 0x7fffu) >= kWinHi;
    }
  }
  over = __reduce_add_sync(0xffffffffu, over);
  if ((threadIdx.x & 31) == 0 && over) reds_add(s.misc + 4u * M_OVER, over);
  __syncthreads();
}

// Descending search over per-thread key ranges: thread t holds `local`, the
// count of keys in [top - PER (t+1), top - PER t), with `above0` keys above
// `top`.  Writes misc[M_BIN / M_ABOVE / M_CNT] for the key where the
// cumulative count reaches kk (M_BIN untouched when it lies outside).
// Two __syncthreads.
template <int PER>
__device__ __forceinline__ void search_desc16(SelArea s, uint32_t local, uint32_t top, uint32_t above0, uint32_t kk) {
  static_assert(PER == 32 || PER == 128, "keys per thread");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // every warp scans its lanes at once; one barrier publishes the warp totals
  uint32_t li = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, li, o);
    if (lane >= o) li += t;
  }
  if (lane == 31) s.set_m(M_WSUM + warp, li);
  __syncthreads();
  const uint4 w0 = lds4(s.misc + 4u * M_WSUM), w1 = lds4(s.misc + 4u * (M_WSUM + 4));
  const uint32_t wt[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
  uint32_t wabove = above0;
#pragma unroll
  for (int q = 0; q < kWarps; ++q) wabove += q < warp ? wt[q] : 0u;
  const uint32_t mine_ex = wabove + li - local;
  const uint32_t own = __ballot_sync(0xffffffffu, (mine_ex < kk) & (kk <= mine_ex + local));
  if (own) {  // this warp holds the owner thread of the k-th key
    const int ol = __ffs(own) - 1;
    const int tb = warp * 32 + ol;
    const uint32_t above = __shfl_sync(0xffffffffu, mine_ex, ol);
    const uint32_t ktop = top - static_cast<uint32_t>(PER) * static_cast<uint32_t>(tb);  // owner's keys: [ktop - PER, ktop)
    constexpr int KL = PER / 32;  // keys per lane, descending from ktop - 1 - KL * lane
    uint32_t c[KL];
    uint32_t lsum = 0;
#pragma unroll
    for (int q = 0; q < KL; ++q) {
      const uint32_t key = ktop - 1u - static_cast<uint32_t>(KL * lane + q);
      c[q] = (lds(s.h16 + 4u * (key >> 1)) >> (16 * (key & 1u))) & 0xffffu;
      lsum += c[q];
    }
    uint32_t linc = lsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, linc, o);
      if (lane >= o) linc += t;
    }
    uint32_t acc = above + linc - lsum;
#pragma unroll
    for (int q = 0; q < KL; ++q) {
      const bool hitq = (acc < kk) & (kk <= acc + c[q]);
      sts_pred(hitq, s.misc + 4u * M_BIN, ktop - 1u - static_cast<uint32_t>(KL * lane + q));
      sts_pred(hitq, s.misc + 4u * M_ABOVE, acc);
      sts_pred(hitq, s.misc + 4u * M_CNT, c[q]);
      acc += c[q];
    }
  }
  __syncthreads();
}

// The exact cut from the 15-bit histogram: the window first (thread t owns
// 32 keys, 4 LDS.128), the whole histogram only if the cut lies outside it
// (thread t owns 128 keys).  Ties at the cut key resolved in ascending index
// order.  Contains __syncthreads.
static __device__ __noinline__ Cut sel_cut16(int n, int k, SelArea s) {
  if (k <= 0) return Cut{0xffffffffu, 0};
  if (k >= n) return Cut{0u, INT_MAX};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t kk = static_cast<uint32_t>(k);
  if (tid == 0) {
    s.set_m(M_TCNT, 0u);
    s.set_m(M_BIN, 0xffffffffu);
  }
  const uint32_t over = s.m(M_OVER);  // published by sel_load16's __syncthreads
  RSP_SEL_STAMP(1);
  if (over < kk) {
    static_assert(kThreads * 32 == static_cast<int>(kWinKeys), "window ownership");
    // threads sit 64 B apart: rotate the chunk order by lane / 2 so each
    // 8-lane phase of an LDS.128 hits 8 distinct bank groups
    const uint32_t base = s.h16 + 4u * ((kWinHi - 32u * static_cast<uint32_t>(tid + 1)) >> 1);
    uint4 u[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) u[q] = lds4(base + 16u * ((q + (lane >> 1)) & 3));
    uint32_t packed = 0;  // counter pairs summed as words: low halves total <= n < 65536
#pragma unroll
    for (int q = 0; q < 4; ++q) packed += u[q].x + u[q].y + u[q].z + u[q].w;
    search_desc16<32>(s, (packed & 0xffffu) + (packed >> 16), kWinHi, over, kk);
  } else {
    __syncthreads();  // M_BIN sentinel visible
  }
  RSP_SEL_STAMP(2);
  if (s.m(M_BIN) == 0xffffffffu) {  // outside the window: the whole histogram
    static_assert(kThreads * 128 == 32768, "15-bit histogram ownership");
    const uint32_t base = s.h16 + 4u * static_cast<uint32_t>(kH16Words - 64 * (tid + 1));
    uint4 u[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) u[q] = lds4(base + 16u * ((q + lane) & 15));
    uint32_t packed = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) packed += u[q].x + u[q].y + u[q].z + u[q].w;
    search_desc16<128>(s, (packed & 0xffffu) + (packed >> 16), 32768u, 0u, kk);
  }
  RSP_SEL_STAMP(4);
  const uint32_t key15 = s.m(M_BIN);
  const uint32_t need = kk - s.m(M_ABOVE), cnt = s.m(M_CNT);
  const uint32_t T = key15 << 16;  // the exact k-th key (fp32 bits, sign cleared)
  if (need == cnt) return Cut{T, INT_MAX};  // every channel of the key is in S
  RSP_SEL_STAMP(8);
  // ties: the `need` lowest indices among the `cnt` channels of key15
  if (cnt <= 32 && (n & 7) == 0) {
    // few channels share the key (the common case): packed-pair equality
    // tests, the rare hits appended to a short list, one warp ranks them
    const int nv = n >> 3;
    for (int v0 = 0; v0 < nv; v0 += 4 * kThreads) {
      uint4 u4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) u4[q] = lds4(s.xs + 16u * static_cast<uint32_t>(min(v0 + q * kThreads + tid, nv - 1)));
      uint32_t hit = 0;  // bit 8q + e: channel 8 v_q + e has the key
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t m = pack8(pair_eq(u4[q].x, key15), pair_eq(u4[q].y, key15), pair_eq(u4[q].z, key15),
                                 pair_eq(u4[q].w, key15));
        hit |= (v0 + q * kThreads + tid < nv ? m : 0u) << (8 * q);
      }
      while (hit) {  // rare
        const int bpos = __ffs(hit) - 1;
        hit &= hit - 1u;
        const uint32_t pos = atoms_add(s.misc + 4u * M_TCNT, 1u);
        sts(s.cand + 4u * pos, static_cast<uint32_t>(8 * (v0 + (bpos >> 3) * kThreads + tid) + (bpos & 7)));
      }
    }
    RSP_SEL_STAMP(6);
    __syncthreads();
    RSP_SEL_STAMP(7);
    if (warp == 0) {
      const uint32_t j = lane < static_cast<int>(cnt) ? lds(s.cand + 4u * lane) : 0xffffffffu;
      uint32_t r4[4] = {0u, 0u, 0u, 0u};  // four independent chains
#pragma unroll
      for (int i = 0; i < 32; ++i) r4[i & 3] += __shfl_sync(0xffffffffu, j, i) < j;
      const uint32_t rank = (r4[0] + r4[1]) + (r4[2] + r4[3]);
      sts_pred((lane < static_cast<int>(cnt)) & (rank == need - 1), s.misc + 4u * M_JLIM, j + 1);
    }
  } else {
    // many ties (e.g. zeros): per-thread contiguous ranges, one block scan
    const int j0 = static_cast<int>(static_cast<uint32_t>(n) * tid / kThreads);
    const int j1 = static_cast<int>(static_cast<uint32_t>(n) * (tid + 1) / kThreads);
    uint32_t mine = 0;
    for (int j = j0; j < j1; ++j) mine += (lds_u16(s.xs + 2u * j) & 0x7fffu) == key15;
    const uint32_t ex = block_excl_scan(mine, s.misc + 4u * M_SCAN, nullptr);
    if (ex < need && need <= ex + mine) {
      uint32_t c = ex;
      for (int j = j0; j < j1; ++j) {
        if ((lds_u16(s.xs + 2u * j) & 0x7fffu) == key15 && ++c == need) {
          s.set_m(M_JLIM, static_cast<uint32_t>(j + 1));
          break;
        }
      }
    }
  }
  __syncthreads();
  RSP_SEL_STAMP(5);
  return Cut{T, static_cast<int>(s.m(M_JLIM))};
}

// Deterministic two-list compaction in one sweep: members of range A
// ([a0, a1), predicate pa) and of range B ([b0, b1), predicate pb), each in
// ascending index order: fa(i, j) / fb(i, j) with i the member's position.
// Warp w sweeps a contiguous run of 32-index chunks of each range.
// Returns the list lengths in *na / *nb (all threads).  Two __syncthreads.
template <class PA, class PB, class FA, class FB>
__device__ __forceinline__ void compact2(SelArea s, int a0, int a1, int b0, int b1, PA&& pa, PB&& pb,
                                         FA&& fa, FB&& fb, int* na, int* nb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ca = (max(0, a1 - a0) + 31) >> 5, cb = (max(0, b1 - b0) + 31) >> 5;
  const int pera = (ca + kWarps - 1) / kWarps, perb = (cb + kWarps - 1) / kWarps;
  const int ca0 = min(ca, warp * pera), ca1 = min(ca, (warp + 1) * pera);
  const int cb0 = min(cb, warp * perb), cb1 = min(cb, (warp + 1) * perb);
  uint32_t cnta = 0, cntb = 0;
#pragma unroll 1
  for (int c = ca0; c < ca1; ++c) {
    const int j = a0 + 32 * c + lane;
    cnta += __popc(__ballot_sync(0xffffffffu, j < a1 && pa(j)));
  }
#pragma unroll 1
  for (int c = cb0; c < cb1; ++c) {
    const int j = b0 + 32 * c + lane;
    cntb += __popc(__ballot_sync(0xffffffffu, j < b1 && pb(j)));
  }
  if (lane == 0) {
    s.set_m(M_LISTA + warp, cnta);
    s.set_m(M_LISTB + warp, cntb);
  }
  __syncthreads();
  const uint32_t wa = lane < kWarps ? s.m(M_LISTA + lane) : 0u;
  const uint32_t wb = lane < kWarps ? s.m(M_LISTB + lane) : 0u;
  uint32_t ia = wa, ib = wb;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t ta = __shfl_up_sync(0xffffffffu, ia, o);
    const uint32_t tb = __shfl_up_sync(0xffffffffu, ib, o);
    if (lane >= o) {
      ia += ta;
      ib += tb;
    }
  }
  uint32_t offa = __shfl_sync(0xffffffffu, ia - wa, warp);
  uint32_t offb = __shfl_sync(0xffffffffu, ib - wb, warp);
  *na = static_cast<int>(__shfl_sync(0xffffffffu, ia, kWarps - 1));
  *nb = static_cast<int>(__shfl_sync(0xffffffffu, ib, kWarps - 1));
  const uint32_t lt = lanemask_lt();
#pragma unroll 1
  for (int c = ca0; c < ca1; ++c) {
    const int j = a0 + 32 * c + lane;
    const bool in = j < a1 && pa(j);
    const uint32_t bal = __ballot_sync(0xffffffffu, in);
    if (in) fa(offa + __popc(bal & lt), j);
    offa += __popc(bal);
  }
#pragma unroll 1
  for (int c = cb0; c < cb1; ++c) {
    const int j = b0 + 32 * c + lane;
    const bool in = j < b1 && pb(j);
    const uint32_t bal = __ballot_sync(0xffffffffu, in);
    if (in) fb(offb + __popc(bal & lt), j);
    offb += __popc(bal);
  }
  __syncthreads();
}


// Membership bits of channels j2, j2 + 1 (j2 even) -- in S when `in_s`, in
// S^c otherwise -- restricted to [lo, hi); `w` returns their raw bf16 pair.
__device__ __forceinline__ uint32_t pair_members16(SelArea s, int j2, int lo, int hi, const Cut& cut, bool in_s,
                                                   uint32_t& w) {
  w = lds(s.xs + 2u * static_cast<uint32_t>(min(j2, (hi - 1) & ~1)));
  uint32_t m_in = 0;
  if (cut.T <= 0x7fff0000u) {  // else S is empty
    const uint32_t t15 = cut.T >> 16;
    const uint32_t gt = t15 < 0x7fffu ? pair_gt(w, t15) : 0u;
    const uint32_t eq = pair_eq(w, t15);
    const int jl = min(max(cut.jlim - j2, 0), 2);
    m_in = ((gt >> 15) & 1u) | ((gt >> 30) & 2u) | ((((eq >> 15) & 1u) | ((eq >> 30) & 2u)) & ((1u << jl) - 1u));
  }
  const int lo_off = min(max(lo - j2, 0), 2), hi_off = min(max(hi - j2, 0), 2);
  const uint32_t range = ((1u << hi_off) - 1u) & ~((1u << lo_off) - 1u);
  return (in_s ? m_in : ~m_in) & range;
}

// compact2 for bf16 activations: S-members of [a0, a1) -> fa(p, i, j, bits),
// S^c-members of [b0, b1) -> fb(p, i, j, bits), each ascending (i = position
// in its list, bits = the fp32 bits of x_j); f is called for both channels of
// a lane with p = membership (write only if p).  2 channels per lane: the
// 64-channel chunks of both ranges are spread over all warps (the lists of
// one CTA are short, so the critical path is one or two chunks per warp);
// positions from two ballots per chunk.  Two __syncthreads.
template <class FA, class FB>
__device__ __forceinline__ void compact2_16(SelArea s, const Cut& cut, int a0, int a1, int b0, int b1, FA&& fa,
                                            FB&& fb, int* na, int* nb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int A0 = a0 & ~1, B0 = b0 & ~1;
  const int ca = a1 > a0 ? (a1 - A0 + 63) >> 6 : 0, cb = b1 > b0 ? (b1 - B0 + 63) >> 6 : 0;
  const int ctot = ca + cb, per = (ctot + kWarps - 1) / kWarps;
  const int c0 = min(ctot, warp * per), c1 = min(ctot, (warp + 1) * per);
  uint32_t w;
  uint32_t cnta = 0, cntb = 0;
#pragma unroll 1
  for (int c = c0; c < c1; ++c) {
    if (c < ca) cnta += __popc(pair_members16(s, A0 + 64 * c + 2 * lane, a0, a1, cut, true, w));
    else cntb += __popc(pair_members16(s, B0 + 64 * (c - ca) + 2 * lane, b0, b1, cut, false, w));
  }
  cnta = __reduce_add_sync(0xffffffffu, cnta);
  cntb = __reduce_add_sync(0xffffffffu, cntb);
  if (lane == 0) {
    s.set_m(M_LISTA + warp, cnta);
    s.set_m(M_LISTB + warp, cntb);
  }
  __syncthreads();
  const uint4 la0 = lds4(s.misc + 4u * M_LISTA), la1 = lds4(s.misc + 4u * (M_LISTA + 4));
  const uint4 lb0 = lds4(s.misc + 4u * M_LISTB), lb1 = lds4(s.misc + 4u * (M_LISTB + 4));
  const uint32_t wa[8] = {la0.x, la0.y, la0.z, la0.w, la1.x, la1.y, la1.z, la1.w};
  const uint32_t wb[8] = {lb0.x, lb0.y, lb0.z, lb0.w, lb1.x, lb1.y, lb1.z, lb1.w};
  uint32_t offa = 0, offb = 0, tota = 0, totb = 0;
#pragma unroll
  for (int q = 0; q < kWarps; ++q) {
    offa += q < warp ? wa[q] : 0u;
    offb += q < warp ? wb[q] : 0u;
    tota += wa[q];
    totb += wb[q];
  }
  *na = static_cast<int>(tota);
  *nb = static_cast<int>(totb);
  const uint32_t lt = lanemask_lt();
  auto emit = [&](int j2, uint32_t m, uint32_t ww, uint32_t& off, auto&& f) {
    const uint32_t bal0 = __ballot_sync(0xffffffffu, m & 1u), bal1 = __ballot_sync(0xffffffffu, (m >> 1) & 1u);
    const uint32_t pre = __popc(bal0 & lt) + __popc(bal1 & lt);
    f((m & 1u) != 0, static_cast<int>(off + pre), j2, ww << 16);
    f((m & 2u) != 0, static_cast<int>(off + pre + (m & 1u)), j2 + 1, ww & 0xffff0000u);
    off += __popc(bal0) + __popc(bal1);
  };
#pragma unroll 1
  for (int c = c0; c < c1; ++c) {
    if (c < ca) {
      const int j2 = A0 + 64 * c + 2 * lane;
      const uint32_t m = pair_members16(s, j2, a0, a1, cut, true, w);
      emit(j2, m, w, offa, fa);
    } else {
      const int j2 = B0 + 64 * (c - ca) + 2 * lane;
      const uint32_t m = pair_members16(s, j2, b0, b1, cut, false, w);
      emit(j2, m, w, offb, fb);
    }
  }
  __syncthreads();
}

}  // namespace rsp
