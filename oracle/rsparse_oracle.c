/*
 * rsparse_oracle.c -- CPU restatement of the R-Sparse linear-operator hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * kernels in paper_2504_19449_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * path (librsparse_b200.so) never links or calls it.
 *
 * Every function restates, in plain C, the reference C++ code it cites
 * (paths relative to the reference tree's proj/core/).  The arithmetic is
 * double precision with the same loop order as the reference, so on the same
 * inputs the results are bit-identical to the reference (pinned against the
 * reference library itself in tests/test_oracle.py via oracle/_ref and the
 * golden fixtures under tests/golden/).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define RSPO_OK 0
#define RSPO_E_USAGE 2

/* ---------------------------------------------------------------------------
 * Seeds and RNG: include/rsparse/rng.hpp:11-76
 * ------------------------------------------------------------------------- */

/* rng.hpp:12-17 */
uint64_t rspo_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* rng.hpp:18-24 */
uint64_t rspo_derive_seed(uint64_t root, const char* tag) {
  uint64_t h = root;
  for (const unsigned char* c = (const unsigned char*)tag; *c; ++c)
    h = rspo_splitmix64(h ^ (uint64_t)(*c));
  return rspo_splitmix64(h);
}

/* std::mt19937_64 (the engine behind rng.hpp:29), restated from its published
 * definition: w=64, n=312, m=156, r=31, a=0xB5026F5AA96619E9, f=6364136223846793005,
 * tempering (u,d)=(29,0x5555555555555555) (s,b)=(17,0x71D67FFFEDA60000)
 * (t,c)=(37,0xFFF7EEE000000000) l=43. */
typedef struct {
  uint64_t mt[312];
  int idx;
  int has_spare;
  double spare;
} rspo_rng;

void rspo_rng_init(rspo_rng* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
  g->has_spare = 0;
  g->spare = 0.0;
}

static void rspo_twist(rspo_rng* g) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  for (int i = 0; i < 312; ++i) {
    uint64_t y = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
    uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
    if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
    g->mt[i] = v;
  }
  g->idx = 0;
}

uint64_t rspo_rng_next_u64(rspo_rng* g) {
  if (g->idx >= 312) rspo_twist(g);
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* rng.hpp:34-36 */
double rspo_rng_uniform01(rspo_rng* g) {
  return (double)(rspo_rng_next_u64(g) >> 11) * 0x1.0p-53;
}

/* rng.hpp:41-50 */
uint64_t rspo_rng_uniform_index(rspo_rng* g, uint64_t n) {
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t v;
  do {
    v = rspo_rng_next_u64(g);
  } while (v >= limit);
  return v % n;
}

/* rng.hpp:53-67: Box-Muller with a cached second value */
double rspo_rng_normal(rspo_rng* g) {
  if (g->has_spare) {
    g->has_spare = 0;
    return g->spare;
  }
  double u1, u2;
  do {
    u1 = rspo_rng_uniform01(g);
  } while (u1 <= 0.0);
  u2 = rspo_rng_uniform01(g);
  const double mag = sqrt(-2.0 * log(u1));
  g->spare = mag * sin(6.283185307179586477 * u2);
  g->has_spare = 1;
  return mag * cos(6.283185307179586477 * u2);
}

/* Fill helpers used by the test fixtures: one Rng(seed), `count` draws. */
void rspo_fill_normal(uint64_t seed, double mean, double stddev, double* out, size_t count) {
  rspo_rng g;
  rspo_rng_init(&g, seed);
  for (size_t i = 0; i < count; ++i) out[i] = mean + stddev * rspo_rng_normal(&g);
}

void rspo_fill_uniform01(uint64_t seed, double* out, size_t count) {
  rspo_rng g;
  rspo_rng_init(&g, seed);
  for (size_t i = 0; i < count; ++i) out[i] = rspo_rng_uniform01(&g);
}

/* ---------------------------------------------------------------------------
 * Selection: src/matrix.cpp:100-117 and src/sparsity.cpp:20-32
 * ------------------------------------------------------------------------- */

typedef struct {
  double mag;
  int64_t idx;
} rspo_key;

/* matrix.cpp:108-113: larger magnitude first, equal magnitudes keep the lower index */
static int rspo_key_cmp(const void* pa, const void* pb) {
  const rspo_key* a = (const rspo_key*)pa;
  const rspo_key* b = (const rspo_key*)pb;
  if (a->mag != b->mag) return a->mag > b->mag ? -1 : 1;
  return (a->idx > b->idx) - (a->idx < b->idx);
}

/* matrix.cpp:100-117.  Writes the k selected indices ascending into out_idx.
 * Returns RSPO_E_USAGE when k > n (matrix.cpp:101-104). */
int rspo_top_k_by_magnitude(const double* x, size_t n, size_t k, int64_t* out_idx) {
  if (k > n) return RSPO_E_USAGE;
  if (k == 0) return RSPO_OK;
  rspo_key* keys = (rspo_key*)malloc(n * sizeof(rspo_key));
  unsigned char* mask = (unsigned char*)calloc(n, 1);
  for (size_t i = 0; i < n; ++i) {
    keys[i].mag = fabs(x[i]);
    keys[i].idx = (int64_t)i;
  }
  qsort(keys, n, sizeof(rspo_key), rspo_key_cmp);
  for (size_t i = 0; i < k; ++i) mask[keys[i].idx] = 1;
  /* matrix.cpp:114-115: resize(k) then sort ascending */
  size_t w = 0;
  for (size_t i = 0; i < n; ++i)
    if (mask[i]) out_idx[w++] = (int64_t)i;
  free(keys);
  free(mask);
  return RSPO_OK;
}

/* sparsity.cpp:26-27: k = ceil(s * n) evaluated in double */
size_t rspo_keep_count(double keep_fraction, size_t n) {
  return (size_t)ceil(keep_fraction * (double)n);
}

/* sparsity.cpp:20-32.  sparse_x (length n) holds x on the kept set, 0 elsewhere;
 * kept (capacity n) receives the ascending kept indices; *k_out their count. */
int rspo_threshold_sparsify(const double* x, size_t n, double keep_fraction, double* sparse_x,
                            int64_t* kept, size_t* k_out) {
  if (!(keep_fraction >= 0.0 && keep_fraction <= 1.0)) return RSPO_E_USAGE;
  const size_t k = rspo_keep_count(keep_fraction, n);
  int st = rspo_top_k_by_magnitude(x, n, k, kept);
  if (st) return st;
  for (size_t i = 0; i < n; ++i) sparse_x[i] = 0.0;
  for (size_t t = 0; t < k; ++t) sparse_x[kept[t]] = x[kept[t]];
  *k_out = k;
  return RSPO_OK;
}

/* ---------------------------------------------------------------------------
 * Operator: src/layer.cpp:74-140, src/matrix.cpp:66-79
 * ------------------------------------------------------------------------- */

/* DecomposedLayer (include/rsparse/layer.hpp:38-48) as plain pointers:
 * w_cols[j*m_out + i] == W(i, j) (layer.hpp:20-27), a_r m_out x r row-major,
 * b_r r x m_in row-major. */
typedef struct {
  size_t m_in, m_out, rank;
  double keep_fraction;
  const double* w_cols;
  const double* a_r;
  const double* b_r;
} rspo_layer;

/* layer.cpp:74-93: y = sum_{j in kept, ascending} x_j * column j.  Adds
 * kept*m*4 to *touched_bytes when non-null (layer.cpp:91). */
int rspo_gather_matvec(const double* w_cols, size_t m_out, size_t m_in, const double* x,
                       const int64_t* kept, size_t nkept, double* y, uint64_t* touched_bytes) {
  for (size_t i = 0; i < m_out; ++i) y[i] = 0.0;
  for (size_t t = 0; t < nkept; ++t) {
    const int64_t j = kept[t];
    if (j < 0 || (size_t)j >= m_in) return RSPO_E_USAGE; /* layer.cpp:83-86 */
    const double xj = x[j];
    const double* col = w_cols + (size_t)j * m_out;
    for (size_t i = 0; i < m_out; ++i) y[i] += xj * col[i];
  }
  if (touched_bytes) *touched_bytes += (uint64_t)nkept * m_out * 4u;
  return RSPO_OK;
}

/* layer.cpp:95-123.  kept_out (capacity m_in, may be NULL) receives the
 * selected channel set so tests can check it against the GPU selector. */
int rspo_forward_ex(const rspo_layer* L, const double* x, double* y, int64_t* kept_out,
                    size_t* k_out) {
  const size_t n = L->m_in, m = L->m_out, r = L->rank;
  double* sparse_x = (double*)malloc((n ? n : 1) * sizeof(double));
  int64_t* kept = (int64_t*)malloc((n ? n : 1) * sizeof(int64_t));
  size_t k = 0;
  int st = rspo_threshold_sparsify(x, n, L->keep_fraction, sparse_x, kept, &k);
  if (st) goto done;
  st = rspo_gather_matvec(L->w_cols, m, n, sparse_x, kept, k, y, NULL);
  if (st) goto done;
  if (r > 0) {
    /* layer.cpp:105-120: residual = x - sparse_x through a_r * b_r */
    double* residual = (double*)malloc(n * sizeof(double));
    double* mid = (double*)malloc(r * sizeof(double));
    for (size_t j = 0; j < n; ++j) residual[j] = x[j] - sparse_x[j];
    for (size_t c = 0; c < r; ++c) {
      const double* row = L->b_r + c * n;
      double acc = 0.0;
      for (size_t j = 0; j < n; ++j) acc += row[j] * residual[j];
      mid[c] = acc;
    }
    for (size_t i = 0; i < m; ++i) {
      const double* row = L->a_r + i * r;
      double acc = 0.0;
      for (size_t c = 0; c < r; ++c) acc += row[c] * mid[c];
      y[i] += acc;
    }
    free(residual);
    free(mid);
  }
  if (kept_out) memcpy(kept_out, kept, k * sizeof(int64_t));
  if (k_out) *k_out = k;
done:
  free(sparse_x);
  free(kept);
  return st;
}

int rspo_forward(const rspo_layer* L, const double* x, double* y) {
  return rspo_forward_ex(L, x, y, NULL, NULL);
}

/* matrix.cpp:66-79: dense row-major y = W x */
void rspo_matvec(const double* w, size_t rows, size_t cols, const double* x, double* y) {
  for (size_t i = 0; i < rows; ++i) {
    const double* row = w + i * cols;
    double acc = 0.0;
    for (size_t j = 0; j < cols; ++j) acc += row[j] * x[j];
    y[i] = acc;
  }
}

/* layer.cpp:125-140 */
void rspo_io_cost(size_t m_in, size_t m_out, double keep_fraction, size_t rank,
                  uint64_t* dense_bytes, uint64_t* touched_bytes, double* relative_cost) {
  const double m = (double)m_out, n = (double)m_in, r = (double)rank;
  const size_t kept_cols = (size_t)ceil(keep_fraction * (double)m_in);
  *dense_bytes = (uint64_t)m_in * m_out * 4u;
  *touched_bytes = ((uint64_t)kept_cols * m_out + (uint64_t)rank * (m_in + m_out)) * 4u;
  *relative_cost = r * (m + n) / (m * n) + keep_fraction;
}

/* src/search.cpp:14-25 (Recipe::rank_for / plan_for) for one layer */
size_t rspo_rank_for(double rho, double budget, size_t m_in, size_t m_out) {
  const double m = (double)m_out, n = (double)m_in;
  const double raw = (1.0 - rho) * budget * (m * n) / (m + n);
  long long r = llround(raw);
  const long long cap = (long long)(m_in < m_out ? m_in : m_out);
  if (r < 0) r = 0;
  if (r > cap) r = cap;
  return (size_t)r;
}

double rspo_keep_fraction_for(double rho, double budget) { return rho * budget; } /* search.hpp:24 */

/* ---------------------------------------------------------------------------
 * Multi-threaded driver for the CPU baseline: independent forwards, one
 * (layer, x) job per work item, `threads` workers.  The reference forward is
 * single-threaded (SURVEY.md §8(b) "Threading"); independent calls are
 * allowed to run concurrently, which is what this does.
 * ------------------------------------------------------------------------- */
typedef struct {
  const rspo_layer* layers;
  const double* const* xs;
  double* const* ys;
  size_t count;
  size_t next;
  pthread_mutex_t mu;
} rspo_pool;

static void* rspo_worker(void* arg) {
  rspo_pool* p = (rspo_pool*)arg;
  for (;;) {
    pthread_mutex_lock(&p->mu);
    size_t i = p->next++;
    pthread_mutex_unlock(&p->mu);
    if (i >= p->count) break;
    rspo_forward(&p->layers[i], p->xs[i], p->ys[i]);
  }
  return NULL;
}

int rspo_forward_many(const rspo_layer* layers, const double* const* xs, double* const* ys,
                      size_t count, int threads) {
  if (threads < 1) threads = 1;
  rspo_pool p = {layers, xs, ys, count, 0, PTHREAD_MUTEX_INITIALIZER};
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) pthread_create(&tids[t], NULL, rspo_worker, &p);
  for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
  free(tids);
  return RSPO_OK;
}
