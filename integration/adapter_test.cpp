// adapter_test.cpp -- the reference-side binding exercised end to end:
// a DecomposedLayer built by the reference's own rsparse::decompose (Jacobi
// SVD, uniform score: layer.cpp:35-72) is uploaded through
// rsparse::b200::Layer and its device forward is compared with the
// reference's rsparse::forward (layer.cpp:95-123) on the same inputs.
// Built by integration/Makefile against /root/reference headers and the
// reference sources compiled in oracle/_ref; run by tests/test_integration.py.
#include <cmath>
#include <cstdio>
#include <vector>

#include "rsparse/layer.hpp"
#include "rsparse/rng.hpp"
#include "rsparse/scores.hpp"
#include "rsparse_b200.hpp"

using namespace rsparse;

static double maxrel(const std::vector<double>& got, const std::vector<double>& want) {
  double num = 0, den = 0;
  for (size_t i = 0; i < want.size(); ++i) {
    num = std::fmax(num, std::fabs(got[i] - want[i]));
    den = std::fmax(den, std::fabs(want[i]));
  }
  return den > 0 ? num / den : num;
}

int main() {
  int failures = 0;
  struct Case { size_t m, n, r; double s; };
  const Case cases[] = {{48, 64, 8, 0.5}, {64, 40, 12, 0.3}, {33, 33, 0, 1.0}, {40, 56, 20, 0.0}};
  for (const Case& c : cases) {
    Rng rng(derive_seed(2504, "adapter"));
    Matrix w(c.m, c.n);
    for (size_t i = 0; i < c.m; ++i)
      for (size_t j = 0; j < c.n; ++j) w(i, j) = rng.normal();
    ScoreMatrix score;
    score.values = Matrix(std::min(c.m, c.n), c.n);
    for (size_t i = 0; i < score.values.rows(); ++i)
      for (size_t j = 0; j < c.n; ++j) score.values(i, j) = 1.0;
    const DecomposedLayer L = decompose(w, SparsityPlan{c.s, c.r}, score);
    std::vector<double> x(c.n);
    for (double& v : x) v = static_cast<float>(rng.normal());  // fp32-exact activations
    const std::vector<double> want = forward(L, x);
    for (rsp_dtype wt : {RSP_F32, RSP_BF16}) {
      b200::Layer dev(L, wt);
      const std::vector<double> got = dev.forward(x);
      const double e = maxrel(got, want);
      const double tol = wt == RSP_F32 ? 1e-5 : 1e-2;
      std::printf("m=%zu n=%zu r=%zu s=%.2f %s: max rel err %.3e (tol %.0e)\n", c.m, c.n, c.r, c.s,
                  wt == RSP_F32 ? "f32" : "bf16", e, tol);
      if (!(e <= tol) || got.size() != want.size()) ++failures;
      // batch of 3 identical tokens == three forwards
      std::vector<double> xs;
      for (int t = 0; t < 3; ++t) xs.insert(xs.end(), x.begin(), x.end());
      const std::vector<double> yb = dev.forward_batch(xs, 3);
      for (int t = 0; t < 3; ++t) {
        std::vector<double> yt(yb.begin() + t * c.m, yb.begin() + (t + 1) * c.m);
        if (!(maxrel(yt, want) <= tol)) ++failures;
      }
    }
    // the reference's error contract: usage_error on a length mismatch
    b200::Layer dev(L, RSP_F32);
    bool threw = false;
    try {
      std::vector<double> bad(c.n + 1, 0.0);
      dev.forward(bad);
    } catch (const usage_error&) {
      threw = true;
    }
    if (!threw) ++failures;
    const rsp_io_report rep = dev.io_cost();
    const IoReport ref = io_cost(L);
    if (rep.dense_bytes != ref.dense_bytes || rep.touched_bytes != ref.touched_bytes ||
        rep.relative_cost != ref.relative_cost)
      ++failures;
  }
  // rank > min(m, n) is the reference's usage_error (layer.cpp:40-44) through the ABI as well
  {
    DecomposedLayer L;
    L.m_in = 4;
    L.m_out = 4;
    L.w_cols.rows = 4;
    L.w_cols.cols = 4;
    L.w_cols.data.assign(16, 1.0);
    L.a_r = Matrix(4, 5);
    L.b_r = Matrix(5, 4);
    L.plan = SparsityPlan{0.5, 5};
    bool threw = false;
    try {
      b200::Layer dev(L, RSP_F32);
    } catch (const usage_error&) {
      threw = true;
    }
    if (!threw) ++failures;
  }
  std::printf(failures ? "ADAPTER FAILED (%d)\n" : "ADAPTER OK\n", failures);
  return failures ? 1 : 0;
}
