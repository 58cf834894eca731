// rsp_internal.h -- host-side launch interface between the C ABI
// (rsp_api.cu) and the sm_100a kernels (rsp_kernels.cu).  Not installed.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace rsp {

// Workspace regions at fixed offsets (shared by every layer using a workspace).
constexpr unsigned kWsBarBytes = 1024;  // {count, gen} + per-column-tile tickets
constexpr unsigned kTAccCap = 2048;     // floats per stage-1 t buffer (r_pad <= 2048)

// Parameters of one fused R-Sparse forward launch (see rsp_kernels.cu).
struct FusedParams {
  const void* Wt;  // [n][m_pad]  input-channel-major W (row j = W[:, j])
  const void* At;  // [r][m_pad]  A_r^T (row c = column c of a_r)
  const void* Bt;  // [n][r_pad]  B_r^T (row j = column j of b_r)
  const void* x;   // [n] fp32 or bf16
  float* y;        // [m] fp32
  float* t_acc;    // [2][kTAccCap] stage-1 sums (fast mode; buffer = barrier generation & 1)
  float* t_part;   // [r_pad][nb_pad] stage-1 partial sums, column b = CTA b (deterministic mode)
  float* y_part;   // [k_splits][m_pad] split-K partial sums (deterministic mode)
  unsigned* bars;  // [2] grid barrier {count, gen} + [col_tiles] tile tickets
  int n, m, m_pad, r, r_pad, k;
  int col_tiles, k_splits;
  int cap_w, cap_u, cap_a;  // per-CTA list capacities (W rows, stage-1 rows, A rows)
  int nb_pad;               // row stride of t_part (grid rounded up to 4)
  int deterministic;        // 1: fixed-order combines (bit-reproducible y)
  int dense;                // 1: all n channels through W, no selection, no low-rank term
  int pdl;                  // 1: launched with programmatic dependent launch
  long long* trace;         // debug: [grid][16] phase timestamps (null in production)
};

struct LaunchPlan {
  int col_tiles = 1, k_splits = 1, grid = 1;
  int cap_w = 1, cap_u = 1, cap_a = 1;
  int nb_pad = 4;
  size_t smem = 0;
  size_t ws_bytes = 0;  // workspace: barriers + t buffers + partials
  size_t ws_acc_off = 0, ws_t_off = 0, ws_y_off = 0;
};

// Shared-memory bytes the fused kernel needs for a plan.
size_t fused_smem_bytes(const LaunchPlan& p, int n, bool x_bf16);

cudaError_t fused_set_smem(size_t smem);
cudaError_t launch_fused(const FusedParams& p, int elem_bytes, bool x_bf16, int grid, size_t smem,
                         cudaStream_t stream, bool pdl);

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
