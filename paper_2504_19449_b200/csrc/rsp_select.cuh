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
// The result is (T, need):  j in S  <=>  key_j > T  or  (key_j == T and
// tie_rank(j) < need), tie_rank(j) = #{i < j : key_i == T}.
//
// Algorithm (one pass over x, no per-pass syncs beyond four):
//   1. load x -> keys in shared memory; shared atomics build a 15-bit
//      histogram of key>>16 (32768 u16 bins packed in 16384 words); the 8-bit
//      coarse histogram of key>>23 is summed from it;
//   2. a 256-entry block scan on the coarse histogram finds the coarse bin
//      holding the k-th largest key; one warp scans that bin's 128 fine bins;
//   3. for bf16 inputs the fine bin IS the key: done.  For fp32 inputs the
//      (usually few) candidates inside the fine bin are ranked by value
//      directly (<= 256), else resolved by two 8-bit radix passes;
//   4. emit: two ballot passes in index order give every element its rank
//      in S or S^c (the tie cut falls out of the tie ballots).
#pragma once

#include <stdint.h>

#include "rsp_device.cuh"

namespace rsp {

constexpr int kFineWords = 16384;  // 32768 15-bit bins as packed u16 pairs
constexpr int kCoarseBins = 256;   // key >> 23
constexpr int kCandMax = 256;
constexpr int kMiscWords = 64;

// misc[] slots
enum : int {
  M_SCAN = 0,       // [0, 17): block-scan scratch
  M_CB = 20,        // coarse bin
  M_NEED1 = 21,
  M_FB = 22,        // fine bin
  M_NEED2 = 23,
  M_CNTFB = 24,
  M_T = 25,
  M_NEED = 26,
  M_CC = 27,        // candidate counter
  M_BIN = 28, M_ABOVE = 29, M_CNT = 30,
  M_WARP = 32,      // [32, 64): per-warp (gt, tie) counts for emit
};

struct SelSmem {
  uint32_t* keys;    // [n] raw fp32 bit patterns of x
  uint32_t* fine;    // [kFineWords]
  uint32_t* coarse;  // [kCoarseBins]
  uint32_t* cand;    // [kCandMax]
  uint32_t* misc;    // [kMiscWords]
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

// Zero the fine histogram (independent of x: may run before griddepcontrol.wait).
__device__ __forceinline__ void sel_clear(const SelSmem& s) {
  uint4* f = reinterpret_cast<uint4*>(s.fine);
  for (int i = threadIdx.x; i < kFineWords / 4; i += kThreads) f[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) s.misc[M_CC] = 0u;
}

// x (fp32 or bf16, any alignment) -> keys[] as fp32 bit patterns.  Vector
// loads when 16-byte aligned.  Ends with __syncthreads.
__device__ __forceinline__ void sel_load(const void* __restrict__ x, bool x_bf16, int n,
                                         const SelSmem& s) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(x);
  if (x_bf16) {
    const uint16_t* xb = static_cast<const uint16_t*>(x);
    if ((a & 15u) == 0 && (n & 7) == 0) {
      const uint4* xv = reinterpret_cast<const uint4*>(x);
      for (int i = threadIdx.x; i < n / 8; i += kThreads) {
        const uint4 u = __ldg(xv + i);
        uint4* d = reinterpret_cast<uint4*>(s.keys + 8 * i);
        d[0] = make_uint4(u.x << 16, u.x & 0xffff0000u, u.y << 16, u.y & 0xffff0000u);
        d[1] = make_uint4(u.z << 16, u.z & 0xffff0000u, u.w << 16, u.w & 0xffff0000u);
      }
    } else {
      for (int j = threadIdx.x; j < n; j += kThreads) s.keys[j] = static_cast<uint32_t>(xb[j]) << 16;
    }
  } else {
    const uint32_t* xf = static_cast<const uint32_t*>(x);
    if ((a & 15u) == 0 && (n & 3) == 0) {
      const uint4* xv = reinterpret_cast<const uint4*>(x);
      uint4* d = reinterpret_cast<uint4*>(s.keys);
      for (int i = threadIdx.x; i < n / 4; i += kThreads) d[i] = __ldg(xv + i);
    } else {
      for (int j = threadIdx.x; j < n; j += kThreads) s.keys[j] = __ldg(xf + j);
    }
  }
  __syncthreads();
}

// 15-bit histogram of key >> 16 (packed u16 shared atomics), then the 8-bit
// coarse histogram key >> 23 as sums of 128 fine bins.  Ends with __syncthreads.
__device__ __forceinline__ void sel_hist(int n, const SelSmem& s) {
  for (int j = threadIdx.x; j < n; j += kThreads) {
    const uint32_t fb = abs_key(s.keys[j]) >> 16;
    atomicAdd(&s.fine[fb >> 1], 1u << ((fb & 1u) * 16u));
  }
  __syncthreads();
  // Two threads per coarse bin, 32 words each, bank-rotated reads.
  const int cbin = threadIdx.x >> 1, half = threadIdx.x & 1;
  const uint32_t* w = s.fine + cbin * 64 + half * 32;
  uint32_t sum = 0;
#pragma unroll 8
  for (int i = 0; i < 32; ++i) {
    const uint32_t v = w[(i + cbin) & 31];
    sum += (v & 0xffffu) + (v >> 16);
  }
  sum += __shfl_xor_sync(0xffffffffu, sum, 1);
  if (half == 0) s.coarse[cbin] = sum;
  __syncthreads();
}

// Descending-bin block search over a 256-bin histogram: returns (bin, count
// above it, its count) for the need-th largest.  All threads participate.
__device__ __forceinline__ void scan256_desc(const uint32_t* hist, uint32_t need, uint32_t* misc) {
  const int tid = threadIdx.x;
  const uint32_t c = tid < 256 ? hist[255 - tid] : 0u;
  const uint32_t above = block_excl_scan(c, misc + M_SCAN, nullptr);
  if (tid < 256 && above < need && need <= above + c) {
    misc[M_BIN] = 255u - tid;
    misc[M_ABOVE] = above;
    misc[M_CNT] = c;
  }
  __syncthreads();
}

__device__ SelResult sel_resolve(int n, int k, bool bf16_keys, const SelSmem& s) {
  if (k <= 0) return SelResult{0xffffffffu, 0u};
  if (k >= n) return SelResult{0u, static_cast<uint32_t>(n)};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t* misc = s.misc;
  // coarse bin
  scan256_desc(s.coarse, static_cast<uint32_t>(k), misc);
  const uint32_t cb = misc[M_BIN];
  const uint32_t need1 = static_cast<uint32_t>(k) - misc[M_ABOVE];
  // fine bin inside cb: bins [cb*128, cb*128+128) = words [cb*64, cb*64+64)
  if (warp == 0) {
    const uint32_t wa = s.fine[cb * 64 + 63 - 2 * lane];  // bins top-4l (hi half), top-4l-1
    const uint32_t wb = s.fine[cb * 64 + 62 - 2 * lane];  // bins top-4l-2, top-4l-3
    const uint32_t c0 = wa >> 16, c1 = wa & 0xffffu, c2 = wb >> 16, c3 = wb & 0xffffu;
    const uint32_t sum = c0 + c1 + c2 + c3;
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t ex = inc - sum;
    if (ex < need1 && need1 <= inc) {
      const uint32_t top = cb * 128 + 127 - 4 * lane;
      const uint32_t cs[4] = {c0, c1, c2, c3};
      uint32_t acc = ex;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (acc + cs[q] >= need1) {
          misc[M_FB] = top - q;
          misc[M_NEED2] = need1 - acc;
          misc[M_CNTFB] = cs[q];
          break;
        }
        acc += cs[q];
      }
    }
  }
  __syncthreads();
  const uint32_t fb = misc[M_FB], need2 = misc[M_NEED2], cntfb = misc[M_CNTFB];
  if (cntfb == need2) return SelResult{(fb << 16) - 1u, 0u};  // whole bin taken (fb > 0 since k < n)
  if (bf16_keys) return SelResult{fb << 16, need2};
  // fp32: rank the candidates (key >> 16 == fb) by their low 16 bits.
  if (cntfb <= static_cast<uint32_t>(kCandMax)) {
    for (int j = tid; j < n; j += kThreads) {
      const uint32_t key = abs_key(s.keys[j]);
      if ((key >> 16) == fb) s.cand[atomicAdd(&misc[M_CC], 1u)] = key & 0xffffu;
    }
    __syncthreads();
    const int c = static_cast<int>(cntfb);
    for (int i = tid; i < c; i += kThreads) {
      const uint32_t v = s.cand[i];
      uint32_t gt = 0, ge = 0;
      for (int q = 0; q < c; ++q) {
        const uint32_t u = s.cand[q];
        gt += u > v;
        ge += u >= v;
      }
      if (gt < need2 && need2 <= ge) {  // every candidate with this value agrees
        misc[M_T] = (fb << 16) | v;
        misc[M_NEED] = need2 - gt;
      }
    }
    __syncthreads();
    return SelResult{misc[M_T], misc[M_NEED]};
  }
  // Many candidates: two 8-bit radix passes over the low 16 bits.
  uint32_t prefix = fb << 16, pmask = 0xffff0000u, need = need2;
  for (int shift = 8; shift >= 0; shift -= 8) {
    for (int i = tid; i < kCoarseBins; i += kThreads) s.coarse[i] = 0u;
    __syncthreads();
    for (int j = tid; j < n; j += kThreads) {
      const uint32_t key = abs_key(s.keys[j]);
      if ((key & pmask) == prefix) atomicAdd(&s.coarse[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    scan256_desc(s.coarse, need, misc);
    need -= misc[M_ABOVE];
    prefix |= misc[M_BIN] << shift;
    pmask |= 255u << shift;
    if (misc[M_CNT] == need) return SelResult{prefix - 1u, 0u};
  }
  return SelResult{prefix, need};
}

// Emit every index with its membership and rank: f(j, bits, in_S, rank),
// rank = position in S (ascending) when in_S, else position in S^c.
// Warp w owns a contiguous range of indices; two ballot passes.  Contains
// one __syncthreads; callers must sync before reading what f wrote.
template <class F>
__device__ __forceinline__ void sel_emit(int n, SelResult r, const SelSmem& s, F&& f) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int chunks = (n + 31) / 32;
  const int per = (chunks + kWarps - 1) / kWarps;
  const int j_lo = min(n, warp * per * 32), j_hi = min(n, (warp + 1) * per * 32);
  uint32_t cgt = 0, ctie = 0;
  for (int base = j_lo; base < j_hi; base += 32) {
    const int j = base + lane;
    const uint32_t key = j < j_hi ? abs_key(s.keys[j]) : 0u;
    cgt += __popc(__ballot_sync(0xffffffffu, j < j_hi && key > r.T));
    ctie += __popc(__ballot_sync(0xffffffffu, j < j_hi && key == r.T));
  }
  if (lane == 0) {
    s.misc[M_WARP + 2 * warp] = cgt;
    s.misc[M_WARP + 2 * warp + 1] = ctie;
  }
  __syncthreads();
  uint32_t tie_before = 0, sel_before = 0;
  for (int w = 0; w < warp; ++w) {
    const uint32_t g = s.misc[M_WARP + 2 * w], t = s.misc[M_WARP + 2 * w + 1];
    const uint32_t take = r.need > tie_before ? min(r.need - tie_before, t) : 0u;
    sel_before += g + take;
    tie_before += t;
  }
  for (int base = j_lo; base < j_hi; base += 32) {
    const int j = base + lane;
    const bool valid = j < j_hi;
    const uint32_t bits = valid ? s.keys[j] : 0u;
    const uint32_t key = abs_key(bits);
    const bool gt = valid && key > r.T;
    const bool tie = valid && key == r.T;
    const uint32_t tmask = __ballot_sync(0xffffffffu, tie);
    const uint32_t trank = tie_before + __popc(tmask & lanemask_lt());
    const bool in = gt || (tie && trank < r.need);
    const uint32_t smask = __ballot_sync(0xffffffffu, in);
    const uint32_t srank = sel_before + __popc(smask & lanemask_lt());
    if (valid) f(j, bits, in, in ? srank : static_cast<uint32_t>(j) - srank);
    tie_before += __popc(tmask);
    sel_before += __popc(smask);
  }
}

}  // namespace rsp
