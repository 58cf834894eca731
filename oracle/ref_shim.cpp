// ref_shim.cpp -- extern "C" access to the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled together with the reference's own
// sources, in place under /root/reference/proj/core/src, by oracle/Makefile
// into oracle/_ref/librsparse_ref.so.  Used to (1) pin the C restatement
// oracle/rsparse_oracle.c, (2) generate the golden fixtures under
// tests/golden/, and (3) time the reference CPU path for bench.py's
// cpu_baseline and `--impl reference` arms.  Never linked by the product.
//
// Nothing here re-implements reference logic: every entry point forwards to
// the reference function named in its comment.
#include <cstdint>
#include <cstring>
#include <atomic>
#include <exception>
#include <span>
#include <thread>
#include <vector>

#include "rsparse/errors.hpp"
#include "rsparse/layer.hpp"
#include "rsparse/matrix.hpp"
#include "rsparse/model.hpp"
#include "rsparse/rng.hpp"
#include "rsparse/scores.hpp"
#include "rsparse/search.hpp"
#include "rsparse/sparsity.hpp"
#include "rsparse/svd.hpp"

using namespace rsparse;

namespace {

int status_of(const std::exception_ptr& e) {
  try {
    std::rethrow_exception(e);
  } catch (const usage_error&) {
    return 2;
  } catch (const numeric_error&) {
    return 1;
  } catch (const io_error&) {
    return 3;
  } catch (...) {
    return 5;
  }
}

#define GUARD(...)                           \
  try {                                      \
    __VA_ARGS__;                             \
    return 0;                                \
  } catch (...) {                            \
    return status_of(std::current_exception()); \
  }

}  // namespace

extern "C" {

// rng.hpp:18-24
uint64_t rspr_derive_seed(uint64_t root, const char* tag) { return derive_seed(root, tag); }

// tests/unit/test_helpers.hpp:12-27 semantics: one Rng(seed), count normal(0, sigma) draws
void rspr_fill_normal(uint64_t seed, double mean, double stddev, double* out, size_t count) {
  Rng rng(seed);
  for (size_t i = 0; i < count; ++i) out[i] = rng.normal(mean, stddev);
}

void rspr_fill_uniform01(uint64_t seed, double* out, size_t count) {
  Rng rng(seed);
  for (size_t i = 0; i < count; ++i) out[i] = rng.uniform01();
}

// matrix.cpp:100-117
int rspr_top_k_by_magnitude(const double* x, size_t n, size_t k, int64_t* out) {
  GUARD({
    auto idx = top_k_by_magnitude(std::span<const double>(x, n), k);
    for (size_t i = 0; i < idx.size(); ++i) out[i] = static_cast<int64_t>(idx[i]);
  })
}

// sparsity.cpp:20-32
int rspr_threshold_sparsify(const double* x, size_t n, double s, double* sparse_x, int64_t* kept,
                            size_t* k_out) {
  GUARD({
    auto [sx, idx] = threshold_sparsify(std::span<const double>(x, n), s);
    std::memcpy(sparse_x, sx.data(), n * sizeof(double));
    for (size_t i = 0; i < idx.size(); ++i) kept[i] = static_cast<int64_t>(idx[i]);
    *k_out = idx.size();
  })
}

// layer.cpp:74-93; w_cols is column-major (data[j*m+i] = W(i,j))
int rspr_gather_matvec(const double* w_cols, size_t m_out, size_t m_in, const double* x,
                       const int64_t* kept, size_t nkept, double* y, uint64_t* touched) {
  GUARD({
    ColMajorMatrix cm;
    cm.rows = m_out;
    cm.cols = m_in;
    cm.data.assign(w_cols, w_cols + m_out * m_in);
    std::vector<size_t> k(kept, kept + nkept);
    auto out = gather_matvec(cm, std::span<const double>(x, m_in), k, touched);
    std::memcpy(y, out.data(), m_out * sizeof(double));
  })
}

// matrix.cpp:66-79
int rspr_matvec(const double* w, size_t rows, size_t cols, const double* x, double* y) {
  GUARD({
    Matrix m(rows, cols, std::vector<double>(w, w + rows * cols));
    auto out = matvec(m, std::span<const double>(x, cols));
    std::memcpy(y, out.data(), rows * sizeof(double));
  })
}

// A DecomposedLayer (layer.hpp:38-48) assembled from host arrays: w_cols
// column-major m_out x m_in, a_r m_out x r row-major, b_r r x m_in row-major.
void* rspr_layer_create(size_t m_in, size_t m_out, size_t rank, double keep_fraction,
                        const double* w_cols, const double* a_r, const double* b_r) {
  try {
    auto* L = new DecomposedLayer();
    L->m_in = m_in;
    L->m_out = m_out;
    L->w_cols.rows = m_out;
    L->w_cols.cols = m_in;
    L->w_cols.data.assign(w_cols, w_cols + m_in * m_out);
    L->a_r = Matrix(m_out, rank, std::vector<double>(a_r, a_r + m_out * rank));
    L->b_r = Matrix(rank, m_in, std::vector<double>(b_r, b_r + rank * m_in));
    L->plan = SparsityPlan{keep_fraction, rank};
    L->selected_components.resize(rank);
    for (size_t c = 0; c < rank; ++c) L->selected_components[c] = c;
    return L;
  } catch (...) {
    return nullptr;
  }
}

void rspr_layer_destroy(void* h) { delete static_cast<DecomposedLayer*>(h); }

// layer.cpp:95-123
int rspr_layer_forward(const void* h, const double* x, double* y) {
  GUARD({
    const auto* L = static_cast<const DecomposedLayer*>(h);
    auto out = forward(*L, std::span<const double>(x, L->m_in));
    std::memcpy(y, out.data(), L->m_out * sizeof(double));
  })
}

// Independent forwards over `threads` std::threads (SPEC.md:331 allows
// concurrent forward calls on immutable layers).  Item i runs
// forward(*layers[i], xs[i]) into ys[i].
int rspr_forward_many(const void* const* layers, const double* const* xs, double* const* ys,
                      size_t count, int threads) {
  if (threads < 1) threads = 1;
  std::atomic<size_t> next{0};
  std::atomic<int> err{0};
  auto work = [&]() {
    for (;;) {
      const size_t i = next.fetch_add(1);
      if (i >= count) break;
      if (int st = rspr_layer_forward(layers[i], xs[i], ys[i])) err = st;
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(work);
  for (auto& t : pool) t.join();
  return err.load();
}

// layer.cpp:125-140
void rspr_io_cost(size_t m_in, size_t m_out, double keep_fraction, size_t rank,
                  uint64_t* dense_bytes, uint64_t* touched_bytes, double* relative_cost) {
  DecomposedLayer L;
  L.m_in = m_in;
  L.m_out = m_out;
  L.plan = SparsityPlan{keep_fraction, rank};
  const IoReport r = io_cost(L);
  *dense_bytes = r.dense_bytes;
  *touched_bytes = r.touched_bytes;
  *relative_cost = r.relative_cost;
}

// search.cpp:14-25
void rspr_plan_for(double rho, double budget, size_t m_in, size_t m_out, double* keep_fraction,
                   size_t* rank) {
  Recipe rec;
  rec.rho = {rho};
  rec.budget = {budget};
  const SparsityPlan p = rec.plan_for(0, m_in, m_out);
  *keep_fraction = p.keep_fraction;
  *rank = p.rank;
}

// layer.cpp:35-72 with a uniform score (test_layer.cpp:19-22), i.e. the
// reference's own Jacobi SVD truncated to `rank` components.  Small shapes
// only (the Jacobi SVD is O(m n^2) per sweep).  Outputs a_r (m x r),
// b_r (r x n) and the selected components (r).
int rspr_decompose_uniform(const double* w, size_t m_out, size_t m_in, double keep_fraction,
                           size_t rank, double* a_r, double* b_r, int64_t* comps) {
  GUARD({
    Matrix W(m_out, m_in, std::vector<double>(w, w + m_out * m_in));
    const size_t kc = std::min(m_out, m_in);
    ScoreMatrix sc{Matrix(kc, m_in, std::vector<double>(kc * m_in, 1.0)), 1, ""};
    const DecomposedLayer L = decompose(W, SparsityPlan{keep_fraction, rank}, sc);
    std::memcpy(a_r, L.a_r.data(), m_out * rank * sizeof(double));
    std::memcpy(b_r, L.b_r.data(), rank * m_in * sizeof(double));
    for (size_t c = 0; c < rank; ++c) comps[c] = static_cast<int64_t>(L.selected_components[c]);
  })
}

// scores.cpp:52-62 (aggregate_scores over score_single_token): tokens[T][n],
// sigma[kc], vt[kc][n] -> scores[kc][n].  num_workers > 1 exercises the
// reference's threaded tree (same result by construction).
int rspr_aggregate_scores(const double* tokens, size_t T, size_t n, const double* sigma, const double* vt,
                          size_t kc, unsigned num_workers, double* scores) {
  GUARD({
    std::vector<std::vector<double>> tok(T);
    for (size_t t = 0; t < T; ++t) tok[t].assign(tokens + t * n, tokens + (t + 1) * n);
    SvdResult svd{Matrix(1, kc), std::vector<double>(sigma, sigma + kc),
                  Matrix(kc, n, std::vector<double>(vt, vt + kc * n))};
    const ScoreMatrix sc = aggregate_scores(tok, svd, "", num_workers);
    std::memcpy(scores, sc.values.data(), kc * n * sizeof(double));
  })
}

// scores.cpp:73-85 (select_components): scores[kc][n] -> comps[r] ascending
int rspr_select_components(const double* scores, size_t kc, size_t n, size_t r, int64_t* comps) {
  GUARD({
    const ScoreMatrix sc{Matrix(kc, n, std::vector<double>(scores, scores + kc * n)), 1, ""};
    const std::vector<size_t> c = select_components(sc, r);
    for (size_t i = 0; i < c.size(); ++i) comps[i] = static_cast<int64_t>(c[i]);
  })
}

// layer.cpp:35-68 (decompose_with_svd) with caller-supplied scores and SVD:
// w[m][n], scores[kc][n], u[m][kc], sigma[kc], vt[kc][n] -> a_r[m][r], b_r[r][n], comps[r]
int rspr_decompose_with_svd(const double* w, size_t m_out, size_t m_in, double keep_fraction, size_t rank,
                            const double* scores, size_t kc, const double* u, const double* sigma,
                            const double* vt, double* a_r, double* b_r, int64_t* comps) {
  GUARD({
    Matrix W(m_out, m_in, std::vector<double>(w, w + m_out * m_in));
    const ScoreMatrix sc{Matrix(kc, m_in, std::vector<double>(scores, scores + kc * m_in)), 1, ""};
    SvdResult svd{Matrix(m_out, kc, std::vector<double>(u, u + m_out * kc)), std::vector<double>(sigma, sigma + kc),
                  Matrix(kc, m_in, std::vector<double>(vt, vt + kc * m_in))};
    const DecomposedLayer L = decompose_with_svd(W, SparsityPlan{keep_fraction, rank}, sc, svd);
    std::memcpy(a_r, L.a_r.data(), m_out * rank * sizeof(double));
    std::memcpy(b_r, L.b_r.data(), rank * m_in * sizeof(double));
    for (size_t c = 0; c < rank; ++c) comps[c] = static_cast<int64_t>(L.selected_components[c]);
  })
}

// model.cpp:115-127 (mlp_forward) over three reference layers made by
// rspr_layer_create: x[n] -> out[n]; hidden width h = up's m_out.
int rspr_mlp_forward(const void* up, const void* gate, const void* down, const double* x, size_t n, double* out) {
  GUARD({
    const auto* U = static_cast<const DecomposedLayer*>(up);
    BlockWeights b;
    b.w_up = Matrix(U->m_out, n);
    const std::vector<double> y = mlp_forward(std::span<const double>(x, n), b, U,
                                              static_cast<const DecomposedLayer*>(gate),
                                              static_cast<const DecomposedLayer*>(down));
    std::memcpy(out, y.data(), y.size() * sizeof(double));
  })
}

// layer.cpp:161-210 (the reference's own fp32 timing harness)
int rspr_bench_matvec(size_t m_in, size_t m_out, double s, size_t reps, uint64_t seed,
                      double* dense_ns, double* gather_ns, uint64_t* dense_bytes,
                      uint64_t* touched_bytes) {
  GUARD({
    const BenchReport r = bench_matvec(m_in, m_out, s, reps, seed);
    *dense_ns = r.dense_ns_median;
    *gather_ns = r.gather_ns_median;
    *dense_bytes = r.dense_bytes;
    *touched_bytes = r.touched_bytes;
  })
}

// layer.cpp:243-267: write a DecomposedLayer (from rspr_layer_create, with
// the given selected components) to an RSPL file.
int rspr_write_layer(void* h, const int64_t* comps, const char* path) {
  GUARD({
    auto* L = static_cast<DecomposedLayer*>(h);
    if (comps)
      for (size_t c = 0; c < L->plan.rank; ++c) L->selected_components[c] = static_cast<size_t>(comps[c]);
    write_decomposed_layer(*L, path);
  })
}

// layer.cpp:269-301: read an RSPL file.  dims = {m_in, m_out, rank};
// w_cols / a_r / b_r / comps may be null (dims only); plan = {s, r}.
int rspr_read_layer(const char* path, uint64_t* dims, double* w_cols, double* a_r, double* b_r,
                    int64_t* comps, double* plan) {
  GUARD({
    const DecomposedLayer L = read_decomposed_layer(path);
    dims[0] = L.m_in;
    dims[1] = L.m_out;
    dims[2] = L.plan.rank;
    if (w_cols) std::memcpy(w_cols, L.w_cols.data.data(), L.w_cols.data.size() * sizeof(double));
    if (a_r) std::memcpy(a_r, L.a_r.data(), L.m_out * L.plan.rank * sizeof(double));
    if (b_r) std::memcpy(b_r, L.b_r.data(), L.plan.rank * L.m_in * sizeof(double));
    if (comps)
      for (size_t c = 0; c < L.plan.rank; ++c) comps[c] = static_cast<int64_t>(L.selected_components[c]);
    if (plan) {
      plan[0] = L.plan.keep_fraction;
      plan[1] = static_cast<double>(L.plan.rank);
    }
  })
}

// -- model-level callers (model.cpp:89-269, search.cpp:36-105) --------------
// init_model + write_model (model.cpp:89-113, 767-792): a reference ToyModel
// in an RSPW file.
int rspr_model_write(size_t num_layers, size_t embed, size_t hidden, size_t heads, size_t vocab, uint64_t seed,
                     size_t max_seq, const char* path) {
  GUARD({
    ModelConfig cfg;
    cfg.num_layers = num_layers;
    cfg.embed_dim = embed;
    cfg.hidden_dim = hidden;
    cfg.num_heads = heads;
    cfg.vocab_size = vocab;
    cfg.seed = seed;
    cfg.max_seq = max_seq;
    write_model(init_model(cfg), path);
  })
}

namespace {
// A DecomposedModel from layer handles (rspr_layer_create), global linear order.
DecomposedModel gather_model(const void* const* layers, size_t count) {
  DecomposedModel dm;
  for (size_t i = 0; i < count; ++i) dm.layers.push_back(*static_cast<const DecomposedLayer*>(layers[i]));
  return dm;
}
}  // namespace

// read_model + model_forward (model.cpp:159-242): logits T x vocab;
// layers == NULL: the dense model.
int rspr_model_logits(const char* path, const int* tokens, size_t T, const void* const* layers, size_t nlayers,
                      size_t decode_start, double* logits) {
  GUARD({
    const ToyModel m = read_model(path);
    DecomposedModel dm;
    if (layers) dm = gather_model(layers, nlayers);
    const Matrix out = model_forward(m, std::span<const int>(tokens, T), layers ? &dm : nullptr, decode_start);
    std::memcpy(logits, out.data(), out.size() * sizeof(double));
  })
}

// read_model + perplexity (model.cpp:244-269).
int rspr_model_perplexity(const char* path, const int* tokens, size_t T, size_t split_point,
                          const void* const* layers, size_t nlayers, double* out) {
  GUARD({
    const ToyModel m = read_model(path);
    DecomposedModel dm;
    if (layers) dm = gather_model(layers, nlayers);
    *out = perplexity(m, std::span<const int>(tokens, T), split_point, layers ? &dm : nullptr);
  })
}

// RecipeEvaluator(model, calibration, seq_len).loss(Recipe{rho, budget}) and
// dense_loss() (search.cpp:36-105): the reference's own pipeline (Jacobi
// SVD, scores, decompose_with_svd, perplexity).
int rspr_recipe_loss(const char* path, const int* calib, size_t ncalib, size_t seq_len, const double* rho,
                     const double* budget, size_t nlin, double* loss, double* dense_loss) {
  GUARD({
    const ToyModel m = read_model(path);
    const RecipeEvaluator ev(m, std::span<const int>(calib, ncalib), seq_len);
    Recipe rc;
    rc.rho.assign(rho, rho + nlin);
    rc.budget.assign(budget, budget + nlin);
    *loss = ev.loss(rc);
    if (dense_loss) *dense_loss = ev.dense_loss();
  })
}

}  // extern "C"
