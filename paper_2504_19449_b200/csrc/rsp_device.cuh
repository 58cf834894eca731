// rsp_device.cuh -- sm_100a device building blocks for the R-Sparse operator:
// PTX wrappers (mbarrier, cp.async.bulk, gpu-scope acquire/release), a
// reusable generation barrier over global memory, block scans, and the
// block-wide exact top-k selector.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rsp {

constexpr int kThreads = 256;               // every kernel in the fused path
constexpr int kWarps = kThreads / 32;

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// The dynamic-smem base as an opaque register value: left to itself nvcc
// rematerializes the shared window base (S2R SR_CgaCtaId + LEA) at every use.
__device__ __forceinline__ uint32_t smem_base_pinned(const void* p) {
  uint32_t v;
  asm volatile("mov.b32 %0, %1;" : "=r"(v) : "r"(smem_u32(p)));
  return v;
}

// Shared-memory accesses through 32-bit shared-window addresses.  Deriving
// a shared address from a generic pointer costs an S2R SR_CgaCtaId that the
// compiler re-issues for every predicated access in a loop (measured: ~130
// cycles per loop iteration in the selector); converting the dynamic smem base
// once and addressing explicitly keeps every access a plain LDS/STS/ATOMS.
__device__ __forceinline__ uint32_t lds(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float ldsf(uint32_t a) { return __uint_as_float(lds(a)); }
__device__ __forceinline__ uint2 lds2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint4 lds4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void stsf(uint32_t a, float v) { sts(a, __float_as_uint(v)); }
__device__ __forceinline__ void sts2(uint32_t a, uint32_t x, uint32_t y) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void sts4(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
// Predicated shared stores: inline asm cannot be predicated by the compiler,
// so `if (p) sts(...)` becomes a branch with a reconvergence barrier per call
// site (measured: tens of cycles each); these compile to a single @p STS.
__device__ __forceinline__ void sts_pred(bool p, uint32_t a, uint32_t v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}" ::"r"(a), "r"(v),
               "r"(static_cast<uint32_t>(p))
               : "memory");
}
__device__ __forceinline__ void sts2_pred(bool p, uint32_t a, uint32_t x, uint32_t y) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q st.shared.v2.u32 [%0], {%1, %2};\n\t}" ::"r"(a),
               "r"(x), "r"(y), "r"(static_cast<uint32_t>(p))
               : "memory");
}
__device__ __forceinline__ uint32_t atoms_add(uint32_t a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void reds_add(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// L2 policy for streamed-once weights.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// 1-D bulk copy global -> this CTA's shared memory, completion counted in
// bytes on `bar` (TMA engine; SASS UBLKCP).  dst/src 16 B aligned, bytes % 16 == 0.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// One 128-byte line into L2 (LSU path; cheap to issue, unlike TMA bulk ops,
// which an SM processes one at a time at ~25 ns each).
__device__ __forceinline__ void prefetch_l2_line(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;"
               : "=r"(old)
               : "l"(p), "r"(v)
               : "memory");
  return old;
}

__device__ __forceinline__ void st_relaxed_gpu(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Reusable generation barrier in global memory: {count, gen}.  One thread per
// CTA calls arrive (after the CTA's writes are fenced) and later wait.  The
// last arriver resets count and publishes gen+1 with release semantics, so the
// words are ready for the next use without any host-side reset.
// ---------------------------------------------------------------------------
// `g` is the generation the caller read before any CTA of this use could
// have arrived (e.g. right after griddepcontrol.wait).
__device__ __forceinline__ void gbar_arrive(unsigned* bar, unsigned expected, unsigned g) {
  __threadfence();
  const unsigned old = atom_add_acq_rel_gpu(bar, 1u);
  if (old == expected - 1) {
    st_relaxed_gpu(bar, 0u);
    st_release_gpu(bar + 1, g + 1);
  }
}

__device__ __forceinline__ void gbar_wait(const unsigned* bar, unsigned g) {
  // Watchdog: a barrier that cannot complete (CTAs not co-resident, corrupted
  // workspace) traps after ~seconds instead of hanging the device.
  unsigned long long spins = 0;
  while (ld_acquire_gpu(bar + 1) == g) {
    __nanosleep(64);
    if (++spins > (1ull << 26)) __trap();
  }
}

// ---------------------------------------------------------------------------
// Block-wide exclusive scan of one u32 per thread (all kThreads threads).
// s_warp: shared address of kWarps scratch words.  Returns the exclusive
// prefix; *total gets the block sum.  Contains two __syncthreads.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t s_warp, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) sts(s_warp + 4u * warp, inc);
  __syncthreads();
  const uint32_t w = lane < kWarps ? lds(s_warp + 4u * lane) : 0u;
  uint32_t wi = w;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
    if (lane >= o) wi += t;
  }
  const uint32_t base = __shfl_sync(0xffffffffu, wi - w, warp);
  if (total) *total = __shfl_sync(0xffffffffu, wi, kWarps - 1);
  __syncthreads();  // the scratch words may be reused right after
  return base + inc - v;
}

// Streaming 16-byte load of weights that are read exactly once per forward
// (no L1 allocation).
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 u;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
               : "l"(p));
  return u;
}

// 16-byte load of data prefetched into L2 (the low-rank A_r rows).
__device__ __forceinline__ uint4 ldg_l2(const void* p) {
  uint4 u;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
               : "l"(p));
  return u;
}

// Ampere-style 16-byte async copy global -> shared (LDGSTS), L2-only.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// mbarrier / bulk-copy helpers on shared-window addresses.
__device__ __forceinline__ void mbar_init_s(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_s(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}
// 1-D TMA bulk copy global -> this CTA's shared memory, completion counted in
// bytes on the mbarrier (dst, src 16-B aligned, bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s_s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// cp.async of 16 bytes to a shared-window address (LDGSTS, L2 only).
__device__ __forceinline__ void cp_async16_s(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16_s_ef(uint32_t dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void named_bar_arrive(int id, int threads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// ---------------------------------------------------------------------------
// 16-byte weight vectors -> fp32 FMAs
// ---------------------------------------------------------------------------
template <typename WT>
struct Vec;

template <>
struct Vec<__nv_bfloat16> {
  static constexpr int kElems = 8;
  __device__ __forceinline__ static void fma(float (&acc)[8], const uint4 u, float c) {
    acc[0] = fmaf(c, __uint_as_float(u.x << 16), acc[0]);
    acc[1] = fmaf(c, __uint_as_float(u.x & 0xffff0000u), acc[1]);
    acc[2] = fmaf(c, __uint_as_float(u.y << 16), acc[2]);
    acc[3] = fmaf(c, __uint_as_float(u.y & 0xffff0000u), acc[3]);
    acc[4] = fmaf(c, __uint_as_float(u.z << 16), acc[4]);
    acc[5] = fmaf(c, __uint_as_float(u.z & 0xffff0000u), acc[5]);
    acc[6] = fmaf(c, __uint_as_float(u.w << 16), acc[6]);
    acc[7] = fmaf(c, __uint_as_float(u.w & 0xffff0000u), acc[7]);
  }
};

template <>
struct Vec<float> {
  static constexpr int kElems = 4;
  __device__ __forceinline__ static void fma(float (&acc)[4], const uint4 u, float c) {
    acc[0] = fmaf(c, __uint_as_float(u.x), acc[0]);
    acc[1] = fmaf(c, __uint_as_float(u.y), acc[1]);
    acc[2] = fmaf(c, __uint_as_float(u.z), acc[2]);
    acc[3] = fmaf(c, __uint_as_float(u.w), acc[3]);
  }
};


// ---------------------------------------------------------------------------
// v3 streaming helpers
// ---------------------------------------------------------------------------
// L2 prefetch that survives the streaming traffic: operands that do not
// depend on x (A_r^T, B_r^T rows) are pulled into L2 while the previous
// linear still runs (under PDL) and read back from L2 later.
__device__ __forceinline__ void prefetch_l2_keep(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}

// Register fence: the value must be materialised here.  Placed after a batch
// of asm-volatile loads it keeps ptxas from interleaving each load with its
// consumer (which leaves one load in flight per warp: measured, streaming
// then runs at a fraction of HBM bandwidth).
__device__ __forceinline__ void reg_fence(uint4& u) {
  asm volatile("" : "+r"(u.x), "+r"(u.y), "+r"(u.z), "+r"(u.w));
}

// Streamed-once weights: no L1 allocation, first in line for L2 eviction.
#ifndef RSP_LDG
#define RSP_LDG 0
#endif
__device__ __forceinline__ uint4 ldg_stream_ef(const void* p, uint64_t pol) {
  uint4 u;
#if RSP_LDG == 1
  asm volatile("ld.global.cg.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
               : "l"(p), "l"(pol));
#elif RSP_LDG == 2
  asm volatile("ld.global.nc.L1::evict_first.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
               : "l"(p), "l"(pol));
#else
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
               : "l"(p), "l"(pol));
#endif
  return u;
}

// Vector float reduction into global memory (sm_90+): no return value,
// performed at L2.  p must be 16-byte aligned.
__device__ __forceinline__ void red_add_v2(float* p, float a, float b) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}
__device__ __forceinline__ void red_add_f32(float* p, float a) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(a) : "memory");
}

__device__ __forceinline__ float ldcg_f32(const float* p) { return __ldcg(p); }


// ---------------------------------------------------------------------------
// Counting barriers on workspace words that start every launch at zero (the
// stack kernel's last CTA resets them): arrive = red.release.gpu (callers
// __syncthreads first so the whole CTA's writes are ordered before it), wait
// = acquire-poll until the count reaches the number of arriving CTAs.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void spin_until_count(const unsigned* p, unsigned target) {
  unsigned long long spins = 0;
  while (ld_acquire_gpu(p) < target) {
    if (++spins > (1ull << 28)) __trap();  // watchdog: CTAs not co-resident / corrupted workspace
  }
}

// ---------------------------------------------------------------------------
// Cross-process exchange counters (row-sharded ranks on several GPUs): 64-bit
// words in every rank's exchange area, mapped into the peers over NVLink.
// They are cumulative (never reset: a late arrival from a slower rank can
// not race a reset), so a wait compares against (launch epoch + 1) x the
// arrivals of one launch.  Publish = fence.acq_rel.sys, then relaxed
// sys-scope adds on every rank's word (one fence for all peers); wait =
// sys-scope acquire poll.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void red_relaxed_sys_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void spin_until_u64_sys(const unsigned long long* p, unsigned long long target) {
  unsigned long long spins = 0;
  while (ld_acquire_sys_u64(p) < target) {
    if (++spins > (1ull << 26)) __trap();  // watchdog: a rank that never launched / arrived
  }
}

}  // namespace rsp
