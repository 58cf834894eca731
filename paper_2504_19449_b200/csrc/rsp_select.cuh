// rsp_select.cuh -- exact block-wide top-k on |x| for one CTA of 512 threads.
//
// Reference semantics (matrix.cpp:100-117, sparsity.cpp:20-32): S = the k
// indices of largest |x|, ties broken toward the LOWER index, reported in
// ascending index order; S^c is the complement, also ascending.
//
// Keys are IEEE-754 fp32 bit patterns with the sign cleared.  For finite
// values their unsigned order equals the order of fabs() on the values
// widened to double (what the reference compares), and +0/-0 share key 0 (the
// reference's fabs(-0.0) == fabs(+0.0) tie, broken by index).  bf16 inputs
// are widened exactly (bits << 16).  NaN keys order above +inf (the
// reference's std::sort on NaN is undefined).
//
// The result is (T, need): T is the exact k-th largest key and
//   j in S  <=>  key_j > T  or  (key_j == T and tie_rank(j) < need),
// tie_rank(j) = #{i < j : key_i == T}  (lower index wins the tie).
//
// Algorithm (per-phase cycle costs are measured by tools/select_probe.cu):
//   1. load x -> keys in shared memory, one shared atomic per element into a
//      12-bit histogram of key >> 19 (exponent + 4 mantissa bits, 16 KB);
//   2. a block scan (8 bins per thread, descending) finds the boundary bin
//      holding the k-th largest key;
//   3. the boundary bin's elements (typically 1-3% of n) are gathered; radix
//      descent over their remaining 19 bits (8/8/3-bit digits, histograms of
//      the candidate list only, one-warp scans) yields the exact T.  More than
//      kCandCap candidates (heavy ties) descend over all keys instead;
//   4. count: ballots give every chunk of 32 indices its (greater, tie) counts;
//      one block scan turns them into per-chunk S offsets (tie cut included);
//   5. emit: a CTA re-visits only the chunks overlapping the rank ranges it
//      owns (binary search on the monotone offsets) and ranks those elements
//      with ballot/popc arithmetic.
// All shared memory is addressed through 32-bit shared-window addresses
// (rsp_device.cuh: lds/sts/atoms_add).
#pragma once

#include <stdint.h>

#include "rsp_device.cuh"

#ifndef RSP_SEL_DEBUG
#define RSP_SEL_DEBUG(level, prefix, need, cnt, extra)
#endif

namespace rsp {

constexpr int kHistBins = 4096;  // key >> 19
constexpr int kCandCap = 1024;
constexpr int kCandWords = kCandCap + 64;  // also holds the per-chunk prefix (n/32 + 1 <= 1025)
constexpr int kMiscWords = 192;

// misc[] word slots
enum : int {
  M_SCAN = 0,  // [0, 16): block-scan scratch
  M_BIN = 20, M_ABOVE = 21, M_CNT = 22,
  M_CC = 25,    // candidate counter
  M_LAST = 31,  // fused kernel: "this CTA combines its column tile"
  M_WARP = 32,  // [32, 64): per-warp (strictly-greater, tie) counts for emit
};

// Shared-window byte addresses of the selector's arrays.
struct SelSmem {
  uint32_t keys;  // [n] u32: raw fp32 bit patterns of x
  uint32_t hist;  // [kHistBins] u32
  uint32_t cand;  // [kCandWords] u32: candidate keys, then per-chunk prefix
  uint32_t misc;  // [kMiscWords] u32
  __device__ __forceinline__ uint32_t key(int j) const { return lds(keys + 4u * j); }
  __device__ __forceinline__ uint32_t m(int slot) const { return lds(misc + 4u * slot); }
  __device__ __forceinline__ void set_m(int slot, uint32_t v) const { sts(misc + 4u * slot, v); }
};

struct SelResult {
  uint32_t T;
  uint32_t need;
};

__device__ __forceinline__ uint32_t abs_key(uint32_t bits) { return bits & 0x7fffffffu; }

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}


// Zero the histogram (independent of x: may run before griddepcontrol.wait).
// Callers __syncthreads before sel_load.
__device__ __forceinline__ void sel_clear(const SelSmem& s) {
  for (int i = threadIdx.x; i < kHistBins / 4; i += kThreads) sts4(s.hist + 16u * i, make_uint4(0, 0, 0, 0));
  if (threadIdx.x == 0) s.set_m(M_CC, 0u);
}

__device__ __forceinline__ void hist_add(const SelSmem& s, uint32_t bits) {
  reds_add(s.hist + 4u * (abs_key(bits) >> 19), 1u);
}

// x (fp32 or bf16, any alignment) -> keys[] as fp32 bit patterns, and the
// 12-bit histogram (needs sel_clear + barrier first; skipped when `hist` is
// false).  All of a thread's 16-byte loads are issued before any is consumed
// (one memory round trip for n <= 16384 bf16 / 8192 fp32).  Ends with
// __syncthreads.
__device__ __forceinline__ void sel_load(const void* __restrict__ x, bool x_bf16, int n,
                                         const SelSmem& s, bool hist) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(x);
  const int per16 = x_bf16 ? 8 : 4;  // elements per 16 B
  if ((a & 15u) == 0 && (n % per16) == 0) {
    const uint4* xv = reinterpret_cast<const uint4*>(x);
    const int nv = n / per16;
    for (int base = 0; base < nv; base += 4 * kThreads) {
      uint4 u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = base + q * kThreads + threadIdx.x;
        u[q] = i < nv ? __ldg(xv + i) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = base + q * kThreads + threadIdx.x;
        if (i >= nv) continue;
        if (x_bf16) {
          const uint4 d0 = make_uint4(u[q].x << 16, u[q].x & 0xffff0000u, u[q].y << 16, u[q].y & 0xffff0000u);
          const uint4 d1 = make_uint4(u[q].z << 16, u[q].z & 0xffff0000u, u[q].w << 16, u[q].w & 0xffff0000u);
          sts4(s.keys + 32u * i, d0);
          sts4(s.keys + 32u * i + 16u, d1);
          if (hist) {
            hist_add(s, d0.x); hist_add(s, d0.y); hist_add(s, d0.z); hist_add(s, d0.w);
            hist_add(s, d1.x); hist_add(s, d1.y); hist_add(s, d1.z); hist_add(s, d1.w);
          }
        } else {
          sts4(s.keys + 16u * i, u[q]);
          if (hist) {
            hist_add(s, u[q].x); hist_add(s, u[q].y); hist_add(s, u[q].z); hist_add(s, u[q].w);
          }
        }
      }
    }
  } else {
    for (int j = threadIdx.x; j < n; j += kThreads) {
      const uint32_t b = x_bf16 ? static_cast<uint32_t>(static_cast<const uint16_t*>(x)[j]) << 16
                                : __ldg(static_cast<const uint32_t*>(x) + j);
      sts(s.keys + 4u * j, b);
      if (hist) hist_add(s, b);
    }
  }
  __syncthreads();
}

// One warp: descending search of a histogram of nb <= 256 bins for the
// need-th largest -> misc[M_BIN/M_ABOVE/M_CNT].  Caller syncs afterwards.
__device__ __forceinline__ void warp_scan_desc(const SelSmem& s, int nb, uint32_t need) {
  const int lane = threadIdx.x & 31;
  const int per = (nb + 31) / 32;  // bins per lane (<= 8)
  uint32_t c[8];
  uint32_t local = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int bin = nb - 1 - (lane * per + q);
    c[q] = (q < per && bin >= 0) ? lds(s.hist + 4u * max(bin, 0)) : 0u;
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
    if (acc < need && need <= acc + c[q]) {
      s.set_m(M_BIN, static_cast<uint32_t>(nb - 1 - (lane * per + q)));
      s.set_m(M_ABOVE, acc);
      s.set_m(M_CNT, c[q]);
    }
    acc += c[q];
  }
}

__device__ __forceinline__ SelResult sel_resolve(int n, int k, bool bf16_keys, const SelSmem& s) {
  if (k <= 0) return SelResult{0xffffffffu, 0u};
  if (k >= n) return SelResult{0u, static_cast<uint32_t>(n)};
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t kk = static_cast<uint32_t>(k);
  // ---- boundary 12-bit bin: thread t owns bins [4088-8t, 4095-8t], descending
  {
    const uint32_t h = s.hist + 4u * ((kHistBins - 8) - 8 * tid);
    const uint4 lo = lds4(h), hi = lds4(h + 16u);
    const uint32_t c[8] = {hi.w, hi.z, hi.y, hi.x, lo.w, lo.z, lo.y, lo.x};
    uint32_t local = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) local += c[q];
    const uint32_t above = block_excl_scan(local, s.misc + 4u * M_SCAN, nullptr);
    if (above < kk && kk <= above + local) {
      uint32_t acc = above;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (acc < kk && kk <= acc + c[q]) {
          s.set_m(M_BIN, static_cast<uint32_t>(kHistBins - 1 - 8 * tid - q));
          s.set_m(M_ABOVE, acc);
          s.set_m(M_CNT, c[q]);
        }
        acc += c[q];
      }
    }
    __syncthreads();
  }
  uint32_t prefix = s.m(M_BIN) << 19, pmask = 0xfff80000u;
  uint32_t need = kk - s.m(M_ABOVE);
  uint32_t cnt = s.m(M_CNT);
  RSP_SEL_DEBUG(0, prefix, need, cnt, 0u);
  if (cnt == need) return SelResult{prefix - 1u, 0u};  // whole bin taken (prefix > 0 since k < n)
  // ---- gather the boundary bin's keys (when they fit)
  const int ncand = static_cast<int>(cnt);
  const bool gathered = cnt <= static_cast<uint32_t>(kCandCap);
  if (gathered) {
    for (int j = tid; j < n; j += kThreads) {
      const uint32_t key = abs_key(s.key(j));
      if ((key & pmask) == prefix) sts(s.cand + 4u * atoms_add(s.misc + 4u * M_CC, 1u), key);
    }
  }
  __syncthreads();  // candidates complete before anyone reads them
  // ---- radix descent over the remaining 19 bits (digits 18..11, 10..3, 2..0);
  // as soon as the surviving candidates fit in one warp they are ranked
  // directly by value (gathered case only).
#pragma unroll 1
  for (int p = 0; p < 4; ++p) {
    if (gathered && cnt <= 32u) {
      if (warp == 0) {
        // compact the survivors into lanes, then count greater / equal values
        const int lane = tid & 31;
        uint32_t mine = 0u, have = 0u;
        for (int i0 = 0; i0 < ncand; i0 += 32) {
          const int i = i0 + lane;
          const uint32_t key = i < ncand ? lds(s.cand + 4u * i) : 0u;
          const bool match = i < ncand && (key & pmask) == prefix;
          const uint32_t bal = __ballot_sync(0xffffffffu, match);
          const uint32_t pos = have + __popc(bal & lanemask_lt());
          // lane `pos` receives this key
#pragma unroll 1
          for (uint32_t bb = bal; bb; bb &= bb - 1) {
            const int src = __ffs(bb) - 1;
            const uint32_t v = __shfl_sync(0xffffffffu, key, src);
            const uint32_t dst = have + __popc(bal & ((1u << src) - 1u));
            if (lane == static_cast<int>(dst)) mine = v;
          }
          (void)pos;
          have += __popc(bal);
        }
        uint32_t gt = 0, ge = 0;
#pragma unroll 1
        for (int q = 0; q < static_cast<int>(have); ++q) {
          const uint32_t o = __shfl_sync(0xffffffffu, mine, q);
          gt += o > mine;
          ge += o >= mine;
        }
        if (lane < static_cast<int>(have) && gt < need && need <= ge) {
          s.set_m(M_BIN, mine);
          s.set_m(M_ABOVE, need - gt);
        }
      }
      __syncthreads();
      return SelResult{s.m(M_BIN), s.m(M_ABOVE)};
    }
    if (p == 3) break;
    const int shift = p == 0 ? 11 : (p == 1 ? 3 : 0), nb = p < 2 ? 256 : 8;
    const uint32_t dmask = static_cast<uint32_t>(nb - 1);
    if (tid < 256) sts(s.hist + 4u * tid, 0u);
    __syncthreads();
    if (gathered) {
      for (int i = tid; i < ncand; i += kThreads) {
        const uint32_t key = lds(s.cand + 4u * i);
        if ((key & pmask) == prefix) reds_add(s.hist + 4u * ((key >> shift) & dmask), 1u);
      }
    } else {
      for (int j = tid; j < n; j += kThreads) {
        const uint32_t key = abs_key(s.key(j));
        if ((key & pmask) == prefix) reds_add(s.hist + 4u * ((key >> shift) & dmask), 1u);
      }
    }
    __syncthreads();
    if (warp == 0) warp_scan_desc(s, nb, need);
    __syncthreads();
    need -= s.m(M_ABOVE);
    prefix |= s.m(M_BIN) << shift;
    pmask |= dmask << shift;
    cnt = s.m(M_CNT);
    RSP_SEL_DEBUG(p + 1, prefix, need, cnt, s.m(M_CC));
    if (cnt == need) return SelResult{prefix - 1u, 0u};  // whole sub-bin taken
    if (bf16_keys && p == 0) return SelResult{prefix, need};  // bits 15..0 are zero: exact
  }
  return SelResult{prefix, need};  // exact key T; `need` of its ties (lowest indices) are in S
}

// Lowest `k` set bits of m.
__device__ __forceinline__ uint32_t lowest_bits(uint32_t m, uint32_t k) {
  if (k >= static_cast<uint32_t>(__popc(m))) return m;
  uint32_t r = 0;
  for (uint32_t i = 0; i < k; ++i) {
    const uint32_t b = m & (0u - m);
    r |= b;
    m ^= b;
  }
  return r;
}

// Per-chunk counts and their exclusive prefix (one block scan).  Chunk c =
// indices [32c, 32c+32).  pk[c] (shared u32 array at s.cand, chunks+1 words)
// = (#keys > T before chunk c) | (#keys == T before chunk c) << 16, so the
// number of S elements before chunk c is lo16 + min(need, hi16).  Counts fit
// 16 bits because n <= 32768.  Contains __syncthreads.
__device__ __forceinline__ void sel_count(int n, SelResult r, const SelSmem& s) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunks = (n + 31) / 32;
  // pass A: per-chunk packed counts (warp w walks chunks w, w+16, ...)
#pragma unroll 4
  for (int c = warp; c < chunks; c += kWarps) {
    const int j = c * 32 + lane;
    const uint32_t key = abs_key(lds(s.keys + 4u * min(j, n - 1)));
    const uint32_t gm = __ballot_sync(0xffffffffu, j < n && key > r.T);
    const uint32_t tm = __ballot_sync(0xffffffffu, j < n && key == r.T);
    if (lane == 0) sts(s.cand + 4u * c, __popc(gm) | (static_cast<uint32_t>(__popc(tm)) << 16));
  }
  __syncthreads();
  // exclusive prefix over chunks: thread t owns chunks 2t, 2t+1
  const int c0 = 2 * threadIdx.x;
  const uint32_t a0 = c0 < chunks ? lds(s.cand + 4u * c0) : 0u;
  const uint32_t a1 = c0 + 1 < chunks ? lds(s.cand + 4u * (c0 + 1)) : 0u;
  uint32_t total;
  const uint32_t ex = block_excl_scan(a0 + a1, s.misc + 4u * M_SCAN, &total);
  if (c0 < chunks) sts(s.cand + 4u * c0, ex);
  if (c0 + 1 < chunks) sts(s.cand + 4u * (c0 + 1), ex + a0);
  if (threadIdx.x == 0) sts(s.cand + 4u * chunks, total);
  __syncthreads();
}

__device__ __forceinline__ uint32_t sel_before(uint32_t pk, uint32_t need) {
  return (pk & 0xffffu) + min(need, pk >> 16);
}

// Emit the elements whose rank in S (in_s) or in S^c (!in_s) lies in
// [lo, hi), ascending rank order: f(j, bits, rank - lo).  Requires sel_count.
// Only the chunks overlapping the rank range are visited (warp-strided).
template <class F>
__device__ __forceinline__ void sel_range_emit(int n, SelResult r, const SelSmem& s, bool in_s,
                                               uint32_t lo, uint32_t hi, F&& f) {
  if (lo >= hi) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunks = (n + 31) / 32;
  // number of (S or S^c) elements before chunk c, monotone in c
  auto before = [&](int c) -> uint32_t {
    const uint32_t sb = sel_before(lds(s.cand + 4u * c), r.need);
    return in_s ? sb : static_cast<uint32_t>(min(32 * c, n)) - sb;
  };
  // first chunk with before(c+1) > lo, last chunk with before(c) < hi
  int a = 0, b = chunks;  // invariant: answer in [a, b)
  while (a + 1 < b) {
    const int mid = (a + b) >> 1;
    if (before(mid) <= lo) a = mid; else b = mid;
  }
  const int c_first = a;
  a = c_first;
  b = chunks;
  while (a + 1 < b) {
    const int mid = (a + b) >> 1;
    if (before(mid) < hi) a = mid; else b = mid;
  }
  const int c_last = a;
  const uint32_t lt = lanemask_lt();
  for (int c = c_first + warp; c <= c_last; c += kWarps) {
    const int j = c * 32 + lane;
    const uint32_t bits = lds(s.keys + 4u * min(j, n - 1));
    const uint32_t key = abs_key(bits);
    const uint32_t gm = __ballot_sync(0xffffffffu, j < n && key > r.T);
    const uint32_t tm = __ballot_sync(0xffffffffu, j < n && key == r.T);
    const uint32_t pk = lds(s.cand + 4u * c);
    const uint32_t tie_pre = pk >> 16;
    const uint32_t take = r.need > tie_pre ? min(r.need - tie_pre, static_cast<uint32_t>(__popc(tm))) : 0u;
    const uint32_t smask = gm | lowest_bits(tm, take);
    const bool in = (smask >> lane) & 1u;
    const uint32_t srank = sel_before(pk, r.need) + __popc(smask & lt);
    const uint32_t rank = in ? srank : static_cast<uint32_t>(j) - srank;
    if (j < n && in == in_s && rank >= lo && rank < hi) f(j, bits, rank - lo);
  }
}

// ===========================================================================
// Fused-kernel selection: static channel ranges + deferred boundary.
//
// The fused kernel never ranks all n channels.  After the 12-bit histogram,
// every channel is classified by its 12-bit bin c = key >> 19 against the
// boundary bin b12 that holds the k-th largest key:
//   c > b12  -> definitely in S;   c < b12 -> definitely in S^c;
//   c == b12 -> boundary (resolved later by one warp: warp_resolve_cut).
// Each CTA compacts only the channel ranges it streams, so W rows can be
// issued right after the histogram scan.
// ===========================================================================
struct Boundary {
  uint32_t b12;   // boundary bin (0xffffffff: S empty)
  uint32_t need;  // boundary-bin members that belong to S
  uint32_t cnt;   // boundary-bin population
  bool all_in;    // the whole boundary bin is in S (cnt == need, or k >= n)
};

__device__ __forceinline__ Boundary sel_boundary(int n, int k, const SelSmem& s) {
  if (k <= 0) return Boundary{0xffffffffu, 0u, 0u, false};
  if (k >= n) return Boundary{0u, 0u, 0u, true};
  const int tid = threadIdx.x;
  const uint32_t kk = static_cast<uint32_t>(k);
  const uint32_t h = s.hist + 4u * ((kHistBins - 8) - 8 * tid);
  const uint4 lo = lds4(h), hi = lds4(h + 16u);
  const uint32_t c[8] = {hi.w, hi.z, hi.y, hi.x, lo.w, lo.z, lo.y, lo.x};
  uint32_t local = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) local += c[q];
  const uint32_t above = block_excl_scan(local, s.misc + 4u * M_SCAN, nullptr);
  if (above < kk && kk <= above + local) {
    uint32_t acc = above;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (acc < kk && kk <= acc + c[q]) {
        s.set_m(M_BIN, static_cast<uint32_t>(kHistBins - 1 - 8 * tid - q));
        s.set_m(M_ABOVE, acc);
        s.set_m(M_CNT, c[q]);
      }
      acc += c[q];
    }
  }
  __syncthreads();
  Boundary b;
  b.b12 = s.m(M_BIN);
  b.need = kk - s.m(M_ABOVE);
  b.cnt = s.m(M_CNT);
  b.all_in = b.cnt == b.need;
  return b;
}

// 0: in S, 1: boundary, 2: in S^c
__device__ __forceinline__ int sel_class(uint32_t key, const Boundary& b) {
  const uint32_t c = key >> 19;
  if (b.b12 == 0xffffffffu) return 2;
  if (c > b.b12 || (c == b.b12 && b.all_in)) return 0;
  return c == b.b12 ? 1 : 2;
}

// Deterministic compaction of channels [lo, hi) by class: f(cls, i, j, bits)
// with i the position among that class's members of the range in ascending
// channel order.  Class totals land in misc[M_CLS + cls].  One barrier.
constexpr int M_CLS = 64;   // [64, 70): class totals (3 per compaction slot)
constexpr int M_CLSW = 72;  // [72, 168): per-warp class counts (48 per slot)
template <class F>
__device__ __forceinline__ void sel_compact(const SelSmem& s, int lo, int hi, const Boundary& b,
                                            int slot, F&& f) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int len = max(0, hi - lo);
  const int chunks = (len + 31) / 32;
  const int per = (chunks + kWarps - 1) / kWarps;
  const int c_lo = min(chunks, warp * per), c_hi = min(chunks, (warp + 1) * per);
  uint32_t cnt[3] = {0u, 0u, 0u};
#pragma unroll 1
  for (int c = c_lo; c < c_hi; ++c) {
    const int j = lo + c * 32 + lane;
    const int cls = j < hi ? sel_class(abs_key(s.key(min(j, hi - 1))), b) : 3;
#pragma unroll
    for (int q = 0; q < 3; ++q) cnt[q] += __popc(__ballot_sync(0xffffffffu, cls == q));
  }
  const uint32_t base = s.misc + 4u * (M_CLSW + slot * 3 * kWarps);
  if (lane < 3) sts(base + 4u * (3 * warp + lane), lane == 0 ? cnt[0] : (lane == 1 ? cnt[1] : cnt[2]));
  __syncthreads();
  uint32_t off[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const uint32_t wc = lane < kWarps ? lds(base + 4u * (3 * lane + q)) : 0u;
    uint32_t inc = wc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    off[q] = __shfl_sync(0xffffffffu, inc - wc, warp);
    if (warp == 0 && lane == kWarps - 1) s.set_m(M_CLS + 3 * slot + q, inc);
  }
  const uint32_t lt = lanemask_lt();
#pragma unroll 1
  for (int c = c_lo; c < c_hi; ++c) {
    const int j = lo + c * 32 + lane;
    const uint32_t bits = s.key(min(j, hi - 1));
    const int cls = j < hi ? sel_class(abs_key(bits), b) : 3;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const uint32_t m = __ballot_sync(0xffffffffu, cls == q);
      if (cls == q) f(q, off[q] + __popc(m & lt), j, bits);
      off[q] += __popc(m);
    }
  }
}

// One warp: the exact cut (T, J) of the reference's total order (|x| desc,
// index asc) inside the boundary bin: its need-th member.  Members are the
// gathered (key, index) pairs at s.cand (gathered = true, cnt pairs) or, when
// they did not fit, every channel of the bin (scanned from keys).  Warp-local
// 8-bit radix steps on the key (then on the index for long ties) until <= 32
// members survive; those are ranked pairwise.  `scratch` = 256 + 64 words of
// shared memory private to the warp.  Result in lanes: (T, J).
__device__ __noinline__ void warp_resolve_cut(const SelSmem& s, int n, const Boundary& bd, bool gathered,
                                                 uint32_t scratch, uint32_t& T_out, uint32_t& J_out) {
  const int lane = threadIdx.x & 31;
  const int src_n = gathered ? static_cast<int>(bd.cnt) : n;
  // fetch member i: (key, index, valid)
  auto fetch = [&](int i, uint32_t& key, uint32_t& idx) -> bool {
    if (gathered) {
      const uint2 e = lds2(s.cand + 8u * i);
      key = e.x;
      idx = e.y;
      return true;
    }
    key = abs_key(s.key(i));
    idx = static_cast<uint32_t>(i);
    return (key >> 19) == bd.b12;
  };
  uint32_t kpre = bd.b12 << 19, kmask = 0xfff80000u;  // key filter
  uint32_t ipre = 0u, imask = 0u;                      // index filter (ties)
  uint32_t need = bd.need, alive = bd.cnt;
  const uint32_t whist = scratch, wbuf = scratch + 4u * 256;
  // key digits 18..11, 10..3, 2..0, then (ascending) index digits 15..8, 7..0
#pragma unroll 1
  for (int step = 0; step < 5 && alive > 32u; ++step) {
    const bool on_key = step < 3;
    const int shift = step == 0 ? 11 : step == 1 ? 3 : step == 2 ? 0 : step == 3 ? 8 : 0;
    const int nb = step == 2 ? 8 : 256;
    const uint32_t dmask = static_cast<uint32_t>(nb - 1);
    for (int i = lane; i < 256; i += 32) sts(whist + 4u * i, 0u);
    __syncwarp();
#pragma unroll 1
    for (int i0 = 0; i0 < src_n; i0 += 32) {
      const int i = i0 + lane;
      uint32_t key = 0, idx = 0;
      const bool ok = i < src_n && fetch(i, key, idx) && (key & kmask) == kpre && (idx & imask) == ipre;
      if (ok) reds_add(whist + 4u * ((on_key ? key : idx) >> shift & dmask), 1u);
    }
    __syncwarp();
    // keys: descending bins (largest first); indices: ascending (lowest first)
    const int per = (nb + 31) / 32;
    uint32_t c[8], local = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int pos = lane * per + q;
      const int bin = on_key ? nb - 1 - pos : pos;
      c[q] = (q < per && pos < nb) ? lds(whist + 4u * bin) : 0u;
      local += c[q];
    }
    uint32_t inc = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    uint32_t acc = inc - local, my_bin = 0, my_above = 0, my_cnt = 0;
    bool found = false;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int pos = lane * per + q;
      if (!found && acc < need && need <= acc + c[q]) {
        found = true;
        my_bin = static_cast<uint32_t>(on_key ? nb - 1 - pos : pos);
        my_above = acc;
        my_cnt = c[q];
      }
      acc += c[q];
    }
    const int src = __ffs(__ballot_sync(0xffffffffu, found)) - 1;
    const uint32_t bin = __shfl_sync(0xffffffffu, my_bin, src);
    need -= __shfl_sync(0xffffffffu, my_above, src);
    alive = __shfl_sync(0xffffffffu, my_cnt, src);
    if (on_key) {
      kpre |= bin << shift;
      kmask |= dmask << shift;
    } else {
      ipre |= bin << shift;
      imask |= dmask << shift;
    }
  }
  // <= 32 survivors: compact into lanes, rank in the total order
  uint32_t have = 0;
#pragma unroll 1
  for (int i0 = 0; i0 < src_n; i0 += 32) {
    const int i = i0 + lane;
    uint32_t key = 0, idx = 0;
    const bool ok = i < src_n && fetch(i, key, idx) && (key & kmask) == kpre && (idx & imask) == ipre;
    const uint32_t bal = __ballot_sync(0xffffffffu, ok);
    if (ok) sts2(wbuf + 8u * (have + __popc(bal & lanemask_lt())), key, idx);
    have += __popc(bal);
  }
  __syncwarp();
  const uint2 me = lane < static_cast<int>(have) ? lds2(wbuf + 8u * lane) : make_uint2(0u, 0xffffffffu);
  uint32_t rank = 0;
  for (int q = 0; q < static_cast<int>(have); ++q) {
    const uint32_t ok = __shfl_sync(0xffffffffu, me.x, q), oi = __shfl_sync(0xffffffffu, me.y, q);
    rank += (ok > me.x) || (ok == me.x && oi < me.y);
  }
  const int who = __ffs(__ballot_sync(0xffffffffu, lane < static_cast<int>(have) && rank == need - 1)) - 1;
  T_out = __shfl_sync(0xffffffffu, me.x, who);
  J_out = __shfl_sync(0xffffffffu, me.y, who);
}

}  // namespace rsp
