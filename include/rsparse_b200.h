/*
 * rsparse_b200.h -- C ABI of the B200-native R-Sparse linear operator.
 *
 * This is the drop-in boundary for the reference's operator API
 * (namespace rsparse, /root/reference/proj/core/include/rsparse/layer.hpp,
 * sparsity.hpp, matrix.hpp, search.hpp).  Each entry point names the
 * reference interface it replaces.  Plain C types only: pointers, sizes and
 * enums -- no torch or C++ types cross this line.  Device pointers are CUDA
 * device addresses on the handle's device; `stream` is a cudaStream_t passed
 * as void*.
 *
 * Errors: every call returns rsp_status.  The codes mirror the reference
 * exception taxonomy (include/rsparse/errors.hpp:8-22): usage_error ->
 * RSP_E_USAGE, numeric_error -> RSP_E_NUMERIC, io_error -> RSP_E_IO; CUDA
 * failures are RSP_E_CUDA.  rsp_last_error() returns the message of the
 * calling thread's last failure.
 *
 * Threading: a handle is immutable after rsp_linear_create (like a
 * DecomposedLayer, layer.hpp:38-48).  rsp_linear_forward is re-entrant
 * across streams when each concurrent call passes its own workspace
 * (SPEC.md:331 allows concurrent forward calls).  rsp_linear_forward_host
 * may be called from several threads on one handle: its per-handle staging
 * buffers are behind a mutex, so such calls run one after another.  A stack
 * owns one workspace: launches of one rsp_stack must be ordered (one stream,
 * or the caller's events); independent tokens use independent stacks.
 */
#ifndef RSPARSE_B200_H_
#define RSPARSE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RSP_ABI_VERSION 3

typedef enum rsp_status {
  RSP_OK = 0,
  RSP_E_NUMERIC = 1, /* rsparse::numeric_error */
  RSP_E_USAGE = 2,   /* rsparse::usage_error   */
  RSP_E_IO = 3,      /* rsparse::io_error      */
  RSP_E_CUDA = 4,    /* CUDA runtime failure   */
  RSP_E_UNSUPPORTED = 5
} rsp_status;

typedef enum rsp_dtype { RSP_F32 = 0, RSP_BF16 = 1, RSP_F64 = 2 } rsp_dtype;

typedef enum rsp_memory { RSP_MEM_HOST = 0, RSP_MEM_DEVICE = 1 } rsp_memory;

/* Layout of desc.w.  ROW_MAJOR is rsparse::Matrix (m_out x m_in, matrix.hpp:13-46);
 * COL_MAJOR is rsparse::ColMajorMatrix::data (data[j*m_out+i] == W(i,j),
 * layer.hpp:20-27), i.e. DecomposedLayer::w_cols. */
typedef enum rsp_w_layout { RSP_W_ROW_MAJOR = 0, RSP_W_COL_MAJOR = 1 } rsp_w_layout;

typedef struct rsp_linear rsp_linear;

/* Everything a rsparse::DecomposedLayer holds (layer.hpp:38-48):
 * W, a_r = U_r sqrt(Sigma_r) (m_out x r row-major), b_r = sqrt(Sigma_r) Vt_r
 * (r x m_in row-major), and its SparsityPlan {keep_fraction, rank}
 * (sparsity.hpp:34-39). */
typedef struct rsp_linear_desc {
  uint32_t m_in;
  uint32_t m_out;
  uint32_t rank;
  double keep_fraction;     /* s in [0,1]; k = ceil(s * m_in) exactly as sparsity.cpp:26-27 */
  int64_t k_override;       /* < 0: use keep_fraction; else explicit k (0..m_in) */
  rsp_dtype weight_dtype;   /* device storage of W, a_r, b_r: RSP_F32 or RSP_BF16 */
  rsp_dtype src_dtype;      /* dtype of the w / a_r / b_r arrays: F64, F32 or BF16 */
  rsp_memory src_memory;    /* where w / a_r / b_r live */
  rsp_w_layout w_layout;
  const void* w;
  const void* a_r;          /* may be NULL when rank == 0 */
  const void* b_r;          /* may be NULL when rank == 0 */
  int device;               /* CUDA ordinal */
  uint32_t shard_rank;      /* output-row sharding: this handle owns rows   */
  uint32_t shard_count;     /* [m_out*rank/count, m_out*(rank+1)/count)     */
  uint32_t flags;           /* RSP_FLAG_* */
} rsp_linear_desc;

/* desc.flags */
#define RSP_FLAG_DETERMINISTIC 1u /* combine split-K partials of y in a fixed order
                                     (bit-reproducible, ~1 us slower per forward);
                                     default: float atomics into y */
#define RSP_FLAG_BATCH_TCGEN05 2u /* batch 2..16: the W / stage-2 products on tcgen05
                                     with TMEM accumulators instead of warp-level
                                     mma.sync (measured slower at B <= 16; default off) */

/* rsp_linear_info.path: which kernels forward() runs (fixed at create). */
#define RSP_PATH_PERSISTENT 1u     /* batch 1: the persistent fused kernel (selection,
                                      gathered rows, low-rank stages in one launch) */
#define RSP_PATH_BATCH_MMA 2u      /* batch 2..16 (bf16 W and x): union-of-masks pass, mma.sync */
#define RSP_PATH_BATCH_TCGEN05 4u  /* batch 2..16: the same pass on tcgen05 / TMEM */
#define RSP_PATH_DETERMINISTIC 8u  /* fixed-order combines (batch > 1 runs per token) */

typedef struct rsp_linear_info {
  uint32_t m_in, m_out, rank, k;
  uint32_t row_begin, row_end; /* output rows owned by this shard */
  uint32_t m_pad, r_pad;       /* padded device widths (multiples of 8) */
  uint32_t col_tiles, k_splits, grid; /* fused-kernel decomposition */
  uint32_t smem_bytes;
  rsp_dtype weight_dtype;
  uint64_t device_bytes;       /* weights + factors resident in HBM */
  uint32_t path;               /* RSP_PATH_* bits: the kernels forward() uses */
} rsp_linear_info;

/* io_cost (layer.cpp:125-140) plus the bytes the B200 kernel actually moves. */
typedef struct rsp_io_report {
  uint64_t dense_bytes;        /* reference: m_in*m_out*4 */
  uint64_t touched_bytes;      /* reference: (ceil(s*n)*m + r*(m+n))*4 */
  double relative_cost;        /* reference: r(m+n)/(mn) + s */
  uint64_t kernel_weight_bytes;/* elem*(k*m + (n-k)*r + r*m), this shard, padded widths */
  uint64_t kernel_total_bytes; /* + x, y, partial-sum traffic */
  uint64_t dense_weight_bytes; /* elem*m*n of this shard (dense GEMV of the same layer) */
} rsp_io_report;

/* -- library ------------------------------------------------------------ */
int rsp_abi_version(void);
const char* rsp_last_error(void);

/* -- plan helpers -------------------------------------------------------- */
/* k = ceil(s * n) evaluated in double (sparsity.cpp:26-27, layer.cpp:129-130). */
rsp_status rsp_keep_count(double keep_fraction, uint32_t n, uint32_t* k_out);
/* Recipe::plan_for for one layer (search.cpp:14-25, search.hpp:24):
 * s = rho*budget, r = clamp(llround((1-rho)*budget*m*n/(m+n)), 0, min(m,n)). */
rsp_status rsp_plan_for(double rho, double budget, uint32_t m_in, uint32_t m_out,
                        double* keep_fraction, uint32_t* rank);

/* Output rows [*begin, *end) owned by shard `shard_rank` of `shard_count`
 * (the row partition rsp_linear_create applies; host-only, no device). */
rsp_status rsp_shard_rows(uint32_t m_out, uint32_t shard_rank, uint32_t shard_count,
                          uint32_t* begin, uint32_t* end);

/* -- operator -------------------------------------------------------------- */
/* Replaces building a rsparse::DecomposedLayer (decompose_with_svd,
 * layer.cpp:35-68, with the factors precomputed on the host).  Uploads W in
 * input-channel-major layout Wt[m_in][m_pad], A_r^T[r][m_pad], B_r^T[m_in][r_pad].
 * Limits of this implementation (RSP_E_UNSUPPORTED, the reference has none):
 * m_in <= 32768 (selection keeps x on chip; above ~28000 channels only with
 * bf16 activations -- fp32 x then returns RSP_E_UNSUPPORTED at forward);
 * one B_r^T row <= 4 KB, i.e.
 * rank <= 2048 with bf16 weights and <= 1024 with fp32 weights (stage-1 t
 * lives in shared memory).  Above rank m*n/(m+n) the factors outweigh W, so
 * the limit only excludes plans slower than the dense GEMV. */
rsp_status rsp_linear_create(const rsp_linear_desc* desc, rsp_linear** out);
void rsp_linear_destroy(rsp_linear* h);
rsp_status rsp_linear_info_get(const rsp_linear* h, rsp_linear_info* out);

/* Bytes of scratch one in-flight forward needs (partial sums + barriers).
 * The buffer must be zeroed once before first use (rsp_workspace_init). */
size_t rsp_linear_workspace_size(const rsp_linear* h, uint32_t batch);
rsp_status rsp_workspace_init(void* workspace, size_t bytes, void* stream);

/* Replaces rsparse::forward(const DecomposedLayer&, span<const double> x)
 * (layer.hpp:75, layer.cpp:95-123).  x_dev: batch x m_in (x_dtype F32/BF16);
 * y_dev: batch x (row_end-row_begin) fp32.  batch 1: one fused kernel
 * (selection, gathered-row GEMV, two-stage low-rank term).  2 <= batch <= 16
 * with bf16 weights and bf16 x: each token keeps its own top-k set (the
 * reference semantics: B independent forwards) and one launch
 * reads the union of the tokens' selected W rows once, on the tensor cores;
 * other combinations run as per-token forwards.  The workspace must be
 * rsp_linear_workspace_size bytes (any batch). */
rsp_status rsp_linear_forward(const rsp_linear* h, const void* x_dev, rsp_dtype x_dtype,
                              float* y_dev, uint32_t batch, void* workspace,
                              size_t workspace_bytes, void* stream);

/* Host-buffer convenience (the end-to-end path): copies x (host) to the
 * device, runs rsp_linear_forward on the handle's internal stream, copies y
 * back and synchronises.  y_host is fp32 (or fp64 when y_dtype == RSP_F64). */
rsp_status rsp_linear_forward_host(rsp_linear* h, const void* x_host, rsp_dtype x_dtype,
                                   void* y_host, rsp_dtype y_dtype, uint32_t batch);

/* Dense baseline of the same layer: y = W x over all m_in channels with the
 * same streaming kernel (k = m_in, no low-rank term).  Reference analogue:
 * the dense sweep of bench_matvec (layer.cpp:142-210) / matvec (matrix.cpp:66-79). */
rsp_status rsp_linear_dense_forward(const rsp_linear* h, const void* x_dev, rsp_dtype x_dtype,
                                    float* y_dev, void* workspace, size_t workspace_bytes,
                                    void* stream);

/* Replaces rsparse::gather_matvec(w_cols, x, kept, touched_bytes)
 * (layer.hpp:69-71, layer.cpp:74-93).  kept_host: nkept indices in
 * accumulation order (validated on the host: out-of-range -> RSP_E_USAGE).
 * Adds nkept*m_out*4 to *touched_bytes when non-NULL (layer.cpp:91). */
rsp_status rsp_gather_matvec(const rsp_linear* h, const void* x_dev, rsp_dtype x_dtype,
                             const int64_t* kept_host, uint32_t nkept, float* y_dev,
                             uint64_t* touched_bytes, void* stream);

/* The channel set forward() selects for x (debug/parity): S ascending into
 * S_host (capacity m_in), *k_out = |S|.  Synchronous. */
rsp_status rsp_linear_selected(const rsp_linear* h, const void* x_dev, rsp_dtype x_dtype,
                               int32_t* S_host, uint32_t* k_out);

/* io_cost (layer.hpp:77, layer.cpp:125-140) plus kernel byte counts. */
rsp_status rsp_linear_io_cost(const rsp_linear* h, rsp_io_report* out);

/* Copy the device-resident operands back as row-major float64
 * (which: 0 = W m_shard x m_in, 1 = a_r m_shard x r, 2 = b_r r x m_in) so a
 * checker can run on exactly the values the kernels read.  Synchronous. */
rsp_status rsp_linear_export(const rsp_linear* h, int which, double* out_host);

/* -- RSPL decomposed-layer files ------------------------------------------------ */
/* The reference's on-disk DecomposedLayer (write_decomposed_layer /
 * read_decomposed_layer, layer.hpp:93-95, layer.cpp:243-301): magic "RSPL",
 * u8 version 1, u32 m_in, m_out, rank, kept width ceil(s*m_in), then f32
 * w_cols (column-major, data[j*m_out+i] = W(i,j)), f32 a_r (m_out x r),
 * f32 b_r (r x m_in), u32 selected components[r], f64 keep_fraction, f64 rank.
 * Little-endian.  Malformed files fail with RSP_E_IO and the reference's
 * io_error message (bad magic, unsupported version, truncated, inconsistent
 * rank fields). */
typedef struct rsp_rspl_header {
  uint32_t m_in, m_out, rank, kept_width;
  double keep_fraction;
} rsp_rspl_header;

/* Host-only parse (no device).  Any array pointer may be NULL (skipped);
 * w_cols holds m_in*m_out, a_r m_out*rank, b_r rank*m_in floats, comps rank. */
rsp_status rsp_rspl_read(const char* path, rsp_rspl_header* header, float* w_cols, float* a_r,
                         float* b_r, uint32_t* comps);

/* read_decomposed_layer + upload: a device-resident operator from an RSPL
 * file.  `opts` (may be NULL) supplies weight_dtype, device, shard_rank,
 * shard_count, flags and k_override; its shape, plan and pointer fields are
 * ignored (they come from the file). */
rsp_status rsp_linear_load_rspl(const char* path, const rsp_linear_desc* opts, rsp_linear** out);

/* write_decomposed_layer of the values the device holds (bf16 handles write
 * their bf16 values widened to f32).  Unsharded handles only. */
rsp_status rsp_linear_save_rspl(const rsp_linear* h, const char* path);

/* The layer's selected SVD components (DecomposedLayer::selected_components):
 * from the RSPL file, else 0..rank-1.  comps holds rank entries. */
rsp_status rsp_linear_components(const rsp_linear* h, uint32_t* comps);

/* -- selector ---------------------------------------------------------------- */
/* Replaces top_k_by_magnitude(span<const double> x, size_t k) (matrix.hpp:63,
 * matrix.cpp:100-117): indices of the k largest |x|, ties to the lower index,
 * ascending.  kept_dev receives k int32 indices; rest_dev (may be NULL)
 * receives the n-k complement indices ascending.  k > n -> RSP_E_USAGE. */
rsp_status rsp_top_k_by_magnitude(const void* x_dev, rsp_dtype x_dtype, uint32_t n, uint32_t k,
                                  int32_t* kept_dev, int32_t* rest_dev, void* stream);

/* Replaces threshold_sparsify(x, s) (sparsity.hpp:43-44, sparsity.cpp:20-32):
 * k = ceil(s*n); sparse_x_dev (fp32, n) = x on the kept set, 0 elsewhere;
 * kept_dev (capacity n) ascending; *k_out = k.  s outside [0,1] -> RSP_E_USAGE. */
rsp_status rsp_threshold_sparsify(const void* x_dev, rsp_dtype x_dtype, uint32_t n,
                                  double keep_fraction, float* sparse_x_dev, int32_t* kept_dev,
                                  uint32_t* k_out, void* stream);

/* -- stack executor ----------------------------------------------------------- */
/* A decode-order sequence of forwards run by ONE persistent kernel launch
 * (captured into a CUDA graph): the instruction working set stays hot across
 * linears and each linear's x-independent operands are prefetched while the
 * previous one drains.  x_devs[i] / y_devs[i] are bound at creation.  By
 * default linear i+1 starts only after linear i's output is complete (its x
 * may be y_i); rsp_stack_create_ex takes wait_prev[i] = 0 for linears that
 * share the previous linear's input (q/k/v, gate/up), which may then overlap.
 * Layers must share device, weight dtype and the deterministic flag. */
typedef struct rsp_stack rsp_stack;
rsp_status rsp_stack_create(const rsp_linear* const* layers, uint32_t count,
                            const void* const* x_devs, rsp_dtype x_dtype, float* const* y_devs,
                            int dense, rsp_stack** out);
rsp_status rsp_stack_create_ex(const rsp_linear* const* layers, uint32_t count,
                               const void* const* x_devs, rsp_dtype x_dtype, float* const* y_devs,
                               int dense, const uint8_t* wait_prev, rsp_stack** out);
/* As rsp_stack_create_ex, with an input operator per linear (x_ops may be
 * NULL = all RSP_XOP_NONE).  RSP_XOP_SILU_GATE: x_devs[i] holds two fp32
 * vectors [a (m_in) | g (m_in)] -- typically the outputs of a stack's up and
 * gate linears written side by side -- and the linear's input is
 * a * silu(g), formed inside the kernel's x load (the gated MLP of
 * model.cpp:115-127: down_proj reads up * silu(gate)); needs x_dtype F32. */
#define RSP_XOP_NONE 0u
#define RSP_XOP_SILU_GATE 1u
rsp_status rsp_stack_create_ops(const rsp_linear* const* layers, uint32_t count,
                                const void* const* x_devs, rsp_dtype x_dtype, float* const* y_devs,
                                int dense, const uint8_t* wait_prev, const uint8_t* x_ops, rsp_stack** out);
/* The general form.  npeer > 1 (row-sharded ranks): the
 * output rows of linear i are written by the kernel to npeer destinations
 * y_peers[i * npeer + p] -- each rank's copy of the FULL y of that linear,
 * offset to this shard's first row -- so the all-gather of y is done by the
 * stores of the producing CTAs themselves instead of a collective after the
 * launch (with several GPUs the destinations are peer-mapped memory over
 * NVLink; on one GPU, several ranks' shards run as one launch over all
 * ranks' buffers).  y_devs is still required (the spans of
 * rsp_stack_launch_host). */
typedef struct rsp_stack_spec {
  const rsp_linear* const* layers;
  uint32_t count;
  const void* const* x_devs;
  rsp_dtype x_dtype;
  float* const* y_devs;
  int dense;
  const uint8_t* wait_prev;  /* may be NULL: every linear waits for its predecessor */
  const uint8_t* x_ops;      /* may be NULL: RSP_XOP_NONE */
  uint32_t npeer;            /* 0 or 1: y_devs only; 2..8: y_peers */
  float* const* y_peers;     /* count x npeer destinations (npeer > 1) */
  uint32_t max_ctas;         /* 0: one CTA per SM; else at most this many CTAs (one per SM), so
                                that independent stacks -- e.g. the B tokens of a small batch,
                                SPEC.md:331 -- run concurrently on disjoint SMs */
  /* Cross-process row sharding (one process per GPU, xrank >= 1 ranks): this
   * rank's stack holds its row shards; y_peers (npeer == xrank) address every
   * rank's y, mapped into this process (rsp_ipc_*), and the group completion
   * counters live in every rank's exchange area: xctr[p] is rank p's area
   * (rsp_stack_exchange_words(count) 64-bit words, zeroed once before the
   * first launch, never reset), xctr[xself] this rank's own.  The CTA that
   * completes a group on its rank publishes the group to all ranks
   * (fence.acq_rel.sys + one add per rank); a dependent group waits for
   * every rank's publication; a start fence per launch
   * keeps a rank from zeroing rows a slower rank still reads.  All ranks must
   * build the same stack (same shapes, even shards: equal per-linear grids,
   * rsp_stack_grids) and launch it the same number of times.  Not with
   * RSP_FLAG_DETERMINISTIC. */
  uint32_t xrank;
  uint32_t xself;
  unsigned long long* const* xctr;
} rsp_stack_spec;
size_t rsp_stack_exchange_words(uint32_t count);
/* Per-linear CTA counts of a stack (count entries): equal on every rank of
 * a cross-process stack. */
rsp_status rsp_stack_grids(const rsp_stack* s, uint32_t* grids, uint32_t count);
rsp_status rsp_stack_create_spec(const rsp_stack_spec* spec, rsp_stack** out);
rsp_status rsp_stack_launch(rsp_stack* s, void* stream);
/* The same launch as a plain kernel launch instead of the stack's own CUDA
 * graph: for callers that capture a larger graph around it (a graph launch
 * inside a stream capture is not capturable everywhere), e.g. the stack
 * launches and NCCL all-gathers of a row-sharded step. */
rsp_status rsp_stack_launch_direct(rsp_stack* s, void* stream);
/* The end-to-end stack path with host buffers: x_host (x_bytes) is copied to
 * the span of device memory covering all the stack's inputs (the x_devs given
 * at creation must lie in one contiguous allocation; x_bytes must equal that
 * span), the stack runs, and the span covering all outputs (y_bytes) is
 * copied to y_host; returns after the stream has synchronised.  Pinned host
 * buffers make both copies asynchronous DMA.  rsp_stack_io_spans reports the
 * two spans. */
rsp_status rsp_stack_io_spans(const rsp_stack* s, size_t* x_bytes, size_t* y_bytes);
rsp_status rsp_stack_launch_host(rsp_stack* s, const void* x_host, size_t x_bytes, void* y_host,
                                 size_t y_bytes, void* stream);
void rsp_stack_destroy(rsp_stack* s);

/* -- peer memory (cross-process exchange) ------------------------------------
 * A device allocation shared between the processes of one node through CUDA
 * IPC: rsp_ipc_alloc (zeroed), rsp_ipc_export its handle (RSP_IPC_HANDLE_BYTES
 * opaque bytes, sent to the peers by the caller), rsp_ipc_open a peer's
 * handle on this process's device (peer access over NVLink), rsp_ipc_close /
 * rsp_ipc_free. */
#define RSP_IPC_HANDLE_BYTES 64
rsp_status rsp_ipc_alloc(int device, size_t bytes, void** dev_ptr);
rsp_status rsp_ipc_free(void* dev_ptr);
rsp_status rsp_ipc_export(const void* dev_ptr, void* handle_out);
rsp_status rsp_ipc_open(int device, const void* handle, void** dev_ptr);
rsp_status rsp_ipc_close(void* dev_ptr);

/* -- diagnostics ---------------------------------------------------------------- */
/* rsp_linear_forward (dense=0) or rsp_linear_dense_forward (dense=1) that also
 * records per-CTA phase timestamps into trace_dev (int64, grid x 16: slot 0 =
 * %globaltimer at CTA start, slots 1..15 = %clock64 cycles since CTA start). */
rsp_status rsp_debug_forward_trace(const rsp_linear* h, const void* x_dev, rsp_dtype x_dtype,
                                   float* y_dev, void* workspace, size_t workspace_bytes,
                                   int64_t* trace_dev, int dense, void* stream);

/* One launch of the stack that records, per (linear l, CTA b), 16 int64 at
 * trace_dev[(l * grid + b) * 16]: [0] %globaltimer at the linear's start,
 * [13] after its dependency wait, [14] at its end, [1..12] %clock64 phase
 * stamps relative to the CTA's start of the linear.  *grid_out = grid. */
rsp_status rsp_debug_stack_trace(rsp_stack* s, int64_t* trace_dev, uint32_t* grid_out, void* stream);
/* Debug: record per-CTA phase clocks in subsequent batched forwards (on != 0). */
rsp_status rsp_debug_set_batch_trace(int on);
/* Debug: per-CTA phase clocks of the last batched forward run with
 * rsp_debug_set_batch_trace(1): host[cta * 16 + phase] (clock64
 * since the CTA started; phases 1 staging, 2 lists, 3 stage 1, 4 arrive,
 * 5 W rows, 6 t barrier, 7 stage 2, 8 combine). */
rsp_status rsp_debug_batch_trace(int64_t* host, uint32_t ctas);

/* -- offline factor build, fp64 device buffers ------------------ */
/* Replaces rsparse::aggregate_scores (scores.cpp:52-62, over score_single_token,
 * scores.cpp:15-29): scores[i][j] = (1/T) sum_t |sigma_i x_tj Vt_ij| for tokens
 * x[T][n], sigma[k], vt[k][n]; the token sum in the reference's pairwise tree,
 * bit-identical.  T == 0 -> RSP_E_USAGE ("requires at least one token"). */
rsp_status rsp_aggregate_scores(const double* tokens, uint32_t T, uint32_t n, const double* sigma,
                                const double* vt, uint32_t k, double* scores, void* stream);
/* Replaces rsparse::select_components (scores.cpp:73-85): the r components of
 * largest score row mass (ties to the lower index), ascending, into comps[r]
 * (device); mass[k] (device) receives the row masses.  r > k -> RSP_E_USAGE. */
rsp_status rsp_select_components(const double* scores, uint32_t k, uint32_t n, uint32_t r, uint32_t* comps,
                                 double* mass, void* stream);
/* The factor split of rsparse::decompose_with_svd (layer.cpp:58-66):
 * a_r[m][r] = U[:, comps] sqrt(sigma[comps]), b_r[r][n] = sqrt(sigma[comps]) Vt[comps, :]
 * (U is m x ucols row-major, Vt is (>= max comps + 1) x n). */
rsp_status rsp_split_factors(const double* u, uint32_t m, uint32_t ucols, const double* sigma, const double* vt,
                             uint32_t n, const uint32_t* comps, uint32_t r, double* a_r, double* b_r, void* stream);
/* Records a layer's selected components (the decompose_with_svd output kept
 * by DecomposedLayer::selected_components; written to RSPL files). */
rsp_status rsp_linear_set_components(rsp_linear* h, const uint32_t* comps, uint32_t r);

/* -- device helpers ------------------------------------------------------------- */
int rsp_device_sm_count(int device);

#ifdef __cplusplus
}
#endif

#endif /* RSPARSE_B200_H_ */
