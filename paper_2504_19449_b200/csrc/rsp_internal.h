// rsp_internal.h -- host-side launch interface between the C ABI
// (rsp_api.cu) and the sm_100a kernels (rsp_kernels.cu).  Not installed.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace rsp {

constexpr unsigned kTAccCap = 2048;  // floats per stage-1 t buffer (r_pad <= 2048)
constexpr unsigned kSlotWords = 32;  // per-linear barrier slot: [0] y arrivals, [1] t arrivals, [2..] tickets
constexpr unsigned kMaxTickets = kSlotWords - 2;
constexpr unsigned kWsHdrBytes = 256;  // [0] launch epoch, [1] CTAs done in this launch
constexpr int kPlanBytes = 96;        // one (linear, CTA) entry of a stack's plan table
constexpr int kMaxPeers = 8;          // y destinations per linear (row-sharded ranks)

// Flags of one linear in a stack launch.
constexpr int kLinWaitPrev = 1;  // its x depends on the previous group's y: wait for that group's CTAs first
constexpr int kLinDense = 2;     // all n channels through W, no selection, no low-rank term
constexpr int kLinSiluGate = 4;  // fp32 x holds [a (n) | g (n)]: the input is a * silu(g) (gated MLP), formed
                                 // in the x load (model.cpp:122-126: hidden = up * silu(gate))

// One linear of a stack launch (descriptors live in device memory; a
// single-linear forward passes its descriptor inline).
struct LinDesc {
  const void* Wt;  // [n][m_pad]  input-channel-major W (row j = W[:, j])
  const void* At;  // [r][m_pad]  A_r^T (row c = column c of a_r)
  const void* Bt;  // [n][r_pad]  B_r^T (row j = column j of b_r)
  const void* x;   // [n] fp32 or bf16
  float* y;        // [m] fp32
  int n, m, m_pad, r, r_pad, k;
  int col_tiles, k_splits, grid;  // CTAs [cta0, cta0 + grid) work on this linear
  int flags;
  int slot;  // index of the linear's barrier slot / t buffers in the workspace
  int cta0;  // first CTA of this linear (linears sharing an input run side by side)
  int dep0, ndep;  // kLinWaitPrev: wait for linears [dep0, dep0 + ndep) (the previous group) to complete
};

// What every CTA needs of every linear to walk the stack without touching its
// full descriptor: membership, dependencies, counter slot (shared memory).
struct LinCtl {
  int flags, dep0, ndep, cta0, grid, slot;
  int aslot;  // slot whose word 0 counts this linear's completed CTAs (shared by its group)
  int garr;   // arrivals that complete the group's counter in one launch (sum of its grids)
};

// Parameters of one launch of the stack kernel (rsp_kernels.cu).
struct StackParams {
  const LinDesc* descs;  // device array of `count` descriptors (null: use `one`)
  LinDesc one;
  int count;
  int n_max, cap_w, cap_u, cap_a;  // shared-memory carve-up (maxima over the linears)
  unsigned* hdr;                   // workspace header
  unsigned* slots;                 // [slots][kSlotWords]
  float* t_acc;                    // [slots][2][kTAccCap] stage-1 sums (parity = launch epoch & 1)
  float* t_part;                   // [r_pad][nb_pad] stage-1 partials (deterministic mode)
  float* y_part;                   // [k_splits][m_pad] split-K partials (deterministic mode)
  int nb_pad;                      // row stride of t_part
  int deterministic;               // 1: fixed-order combines (bit-reproducible y); linears serialised
  int pdl;                         // 1: launched with programmatic dependent launch
  unsigned zero;                   // always 0: a value the compiler cannot fold (load batching in stream_list)
  float* const* ypeer;             // npeer > 1: [count][kMaxPeers] destinations of each linear's y rows
  int npeer;                       // destinations per y (1: the descriptor's y only)
  // Cross-process row sharding (xrank > 0, one launch per rank and token):
  // every rank's exchange words ([xslots] group arrivals + 1 start fence),
  // this rank's own words, the rank count.  Arrivals go to every rank;
  // dependency waits poll the local words (targets x xrank, cumulative).
  unsigned long long* const* xctr;
  unsigned long long* xlocal;
  int xrank, xslots;
  long long* trace;                // debug: [grid][16] phase timestamps of the last linear (null in production)
  const void* plans;               // [count][grid] per-CTA plans (plan_kernel), or null: computed in the kernel
  const LinCtl* ctl;               // [count] control table, or null (single linear: built from `one`)
};

// Workspace byte layout for `slots` linears; t_part/y_part sized for the
// deterministic mode of the largest linear.
struct WsLayout {
  size_t slots_off, tacc_off, tpart_off, ypart_off, bytes;
  static WsLayout make(int slots, int nb_pad, int r_pad_max, int ks_max, int m_pad_max) {
    auto up = [](size_t v) { return (v + 255) / 256 * 256; };
    WsLayout w;
    w.slots_off = kWsHdrBytes;
    w.tacc_off = up(w.slots_off + static_cast<size_t>(slots) * kSlotWords * 4);
    w.tpart_off = up(w.tacc_off + static_cast<size_t>(slots) * 2 * kTAccCap * 4);
    w.ypart_off = up(w.tpart_off + static_cast<size_t>(nb_pad) * (r_pad_max > 8 ? r_pad_max : 8) * 4);
    w.bytes = up(w.ypart_off + static_cast<size_t>(ks_max) * m_pad_max * 4);
    return w;
  }
};

// Shared-memory bytes of the stack kernel for these maxima.
size_t stack_smem_bytes(int n_max, bool x_bf16, int cap_w, int cap_u, int cap_a, int count = 1);

cudaError_t stack_set_smem(size_t smem);
// Fill a stack's plan table (count x grid entries of kPlanBytes) from its device descriptors.
cudaError_t launch_plans(const LinDesc* descs, int count, int grid, int acap, int elem_bytes, void* out,
                         cudaStream_t stream);
// Bytes of the stack kernel's dead x + histogram area (A_r^T row copies).
int stack_acopy_bytes(int n_max, bool x_bf16, int cap_w, int cap_u, int cap_a, int count);
cudaError_t launch_stack(const StackParams& p, int elem_bytes, bool x_bf16, int grid, size_t smem,
                         cudaStream_t stream, bool pdl);

// Batch > 1 forward of one linear (rsp_batch.cu): bf16 W and x, B <= kBatchMax.
constexpr int kBatchMax = 16;
struct BatchParams {
  const void* Wt;   // bf16 [n][m_pad]
  const void* At;   // bf16 [r][m_pad]
  const void* Bt;   // bf16 [n][r_pad]
  const void* x;    // bf16 [B][n]
  float* y;         // fp32 [B][m]  (zero on entry when ks > 1 and !zero_y)
  int2* cuts;       // [B] per-token cuts (workspace)
  float* t_acc;     // [B][r_pad] (workspace; zero on entry, left zero)
  unsigned* ctr;    // [0] t arrivals, [1] CTAs done, [2] cuts published (workspace; zero on entry, left zero)
  int n, m, m_pad, r, r_pad, k, B;
  int cw, ks, grid;  // 64 x cw output columns per CTA, ks channel splits, grid = tiles x ks
  int range_max, slice_max, na_max;  // shared-memory carve-up
  int trace;                         // debug: per-CTA phase clocks into g_batch_trace
  int tc;                            // W / stage-2 products on tcgen05 (cw == 8)
  int zero_y;                        // the kernel zeroes y before the t barrier (ks > 1, low-rank term)
  int pdl;                           // launched with programmatic stream serialization
  unsigned zero;                     // 0, opaque to the compiler (selector load batching)
};
cudaError_t batch_trace_copy(long long* host, int count);

// Offline factor build (rsp_offline.cu), fp64.
cudaError_t launch_scores(const double* x, uint32_t T, uint32_t n, const double* sigma, const double* vt, uint32_t k,
                          double* out, cudaStream_t s);
cudaError_t launch_select_components(const double* scores, uint32_t k, uint32_t n, uint32_t r, uint32_t* comps,
                                     double* mass, cudaStream_t s);
cudaError_t launch_split_factors(const double* u, uint32_t m, uint32_t ucols, const double* sigma, const double* vt,
                                 uint32_t n, const uint32_t* comps, uint32_t r, double* a_r, double* b_r,
                                 cudaStream_t s);
constexpr size_t kBatchWsBytes(int r_pad) { return 512 + static_cast<size_t>(kBatchMax) * r_pad * 4; }
size_t batch_smem_bytes(const BatchParams& p);
cudaError_t launch_batch(const BatchParams& p, bool x_bf16, cudaStream_t stream);

// Stand-alone selector: one CTA.  Any of kept/rest/sparse may be null.
size_t select_smem_bytes(int n, bool x_bf16);
cudaError_t launch_select(const void* x, bool x_bf16, int n, int k, int32_t* kept, int32_t* rest,
                          float* sparse_x, cudaStream_t stream);

// y[i] = sum_t x[kept[t]] * Wt[kept[t]][i], t ascending (gather_matvec).
cudaError_t launch_gather(const void* Wt, int elem_bytes, int m, int m_pad, const void* x,
                          bool x_bf16, const int32_t* kept, int nkept, float* y,
                          cudaStream_t stream);

// dst[c][r] = convert(src[r][c])  (transpose=1) or dst[r][c] = convert(src[r][c]).
// src: rows x cols with leading dimension src_ld, dtype 0=f32 1=bf16 2=f64;
// dst: elem 4 (f32) or 2 (bf16) with leading dimension dst_ld.
cudaError_t launch_convert(const void* src, int src_dtype, size_t rows, size_t cols, size_t src_ld,
                           void* dst, int dst_elem, size_t dst_ld, bool transpose,
                           cudaStream_t stream);

}  // namespace rsp
