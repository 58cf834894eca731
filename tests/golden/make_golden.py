"""Generate tests/golden/golden.npz from the REFERENCE library itself.

Run in the build container (needs oracle/_ref/librsparse_ref.so, i.e. the
reference sources compiled in place by oracle/Makefile):

    python tests/golden/make_golden.py

Every array comes out of the unmodified reference code (rsparse::Rng,
top_k_by_magnitude, threshold_sparsify, decompose (Jacobi SVD, uniform
score), gather_matvec, forward, io_cost, Recipe::plan_for).  The cases
restate the reference unit tests' known-answer inputs and seeds
(tests/unit/test_linalg.cpp:70-106, test_sparsity.cpp:25-76,
test_layer.cpp:92-215) plus tie-heavy and ragged extras.  The fixtures
travel to the GPU box (the reference tree does not).
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import ref_oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def main():
    R = ref_oracle()
    g = {}

    # --- rng.hpp bit-stability -------------------------------------------------
    g["rng.seed42.normal"] = R.normal(42, 64)
    g["rng.seed7.uniform01"] = R.uniform01(7, 64)
    g["rng.derive_seed"] = np.array([R.derive_seed(0, "cfg0.w"), R.derive_seed(42, "cfg1.x"),
                                     R.derive_seed(2**63 + 5, "search")], dtype=np.uint64)

    # --- top_k_by_magnitude KATs (test_linalg.cpp:70-106) -----------------------
    topk = []
    def add_topk(name, x, k):
        x = np.asarray(x, dtype=np.float64)
        try:
            idx = R.top_k_by_magnitude(x, k)
            err = 0
        except Exception:
            idx, err = np.zeros(0, dtype=np.int64), 2
        g[f"topk.{name}.x"] = x
        g[f"topk.{name}.k"] = np.array([k])
        g[f"topk.{name}.idx"] = idx
        g[f"topk.{name}.err"] = np.array([err])
        topk.append(name)

    add_topk("worked", [0.1, -2.0, 0.5, -0.3], 2)
    add_topk("k0", [1.0, 2.0, 3.0], 0)
    add_topk("kn", [1.0, 2.0, 3.0], 3)
    add_topk("k_gt_n", [1.0, 2.0, 3.0], 4)
    add_topk("ties_k1", [1.0, -1.0, 1.0], 1)
    add_topk("ties_k2", [1.0, -1.0, 1.0], 2)
    x40 = R.normal(10, 40)  # random_vector(40, 10)
    for k in range(0, 41, 5):
        add_topk(f"nest40_k{k}", x40, k)
    add_topk("signed_zero", [0.0, -0.0, 0.0, -0.0, 1.0, -0.0], 3)
    add_topk("all_equal", [0.5] * 37, 11)
    add_topk("sign_dups", [3.0, -3.0, 2.0, -2.0, 3.0, 1.0, -1.0, 2.0], 4)
    levels = np.round(R.normal(123, 1000) * 2) / 2  # few distinct levels, heavy ties
    add_topk("levels1000_k500", levels, 500)
    add_topk("levels1000_k137", levels, 137)
    g["topk.names"] = np.array(topk)

    # --- threshold_sparsify KATs (test_sparsity.cpp:25-76) -----------------------
    thr = []
    def add_thr(name, x, s):
        x = np.asarray(x, dtype=np.float64)
        try:
            sx, kept = R.threshold_sparsify(x, s)
            err = 0
        except Exception:
            sx, kept, err = np.zeros(0), np.zeros(0, dtype=np.int64), 2
        g[f"thr.{name}.x"] = x
        g[f"thr.{name}.s"] = np.array([s])
        g[f"thr.{name}.sx"] = sx
        g[f"thr.{name}.kept"] = kept
        g[f"thr.{name}.err"] = np.array([err])
        thr.append(name)

    add_thr("worked", [0.1, -2.0, 0.5, -0.3], 0.5)
    add_thr("s1", [0.3, -0.7, 1.1], 1.0)
    add_thr("s0", [0.3, -0.7, 1.1], 0.0)
    add_thr("s_neg", [0.3, -0.7, 1.1], -0.1)
    add_thr("s_big", [0.3, -0.7, 1.1], 1.5)
    x37 = R.normal(5, 37)  # random_vector(37, 5)
    for s in (0.1, 0.33, 0.5, 0.77, 0.99):
        add_thr(f"n37_s{s}", x37, s)
    g["thr.names"] = np.array(thr)

    # --- forward / gather through reference-decomposed layers --------------------
    fwd = []
    def add_fwd(name, m, n, s, r, wseed, xseeds, quantize_x=False):
        w = R.normal(wseed, m * n).reshape(m, n)  # random_matrix(m, n, wseed)
        a, b, comps = R.decompose_uniform(w, s, r)
        g[f"fwd.{name}.w"] = w
        g[f"fwd.{name}.a_r"] = a
        g[f"fwd.{name}.b_r"] = b
        g[f"fwd.{name}.plan"] = np.array([s, r], dtype=np.float64)
        xs, ys, kepts = [], [], []
        for xs_seed in xseeds:
            x = R.normal(xs_seed, n)
            if quantize_x:
                x = np.round(x * 2.0) / 2.0
            xs.append(x)
            ys.append(R.forward(w.T, a, b, s, x))  # w.T: column-major w_cols data as (n, m)
            kepts.append(R.threshold_sparsify(x, s)[1])
        g[f"fwd.{name}.x"] = np.stack(xs)
        g[f"fwd.{name}.y"] = np.stack(ys)
        for i, kk in enumerate(kepts):
            g[f"fwd.{name}.kept{i}"] = kk
        g[f"fwd.{name}.dense_y"] = np.stack([R.matvec(w, x) for x in xs])
        fwd.append(name)

    add_fwd("dense_s1_r0", 14, 11, 1.0, 0, 66, [67])           # test_layer.cpp:92-97
    add_fwd("factors_s0_rmin", 14, 11, 0.0, 11, 68, [69])      # :99-104
    add_fwd("two_term_64", 64, 64, 0.5, 8, 70, [72, 73, 74])   # :106-117
    add_fwd("split_20x24", 20, 24, 0.25, 5, 75, [77])          # :119-134
    add_fwd("zero_s0_r0", 5, 7, 0.0, 0, 78, [79])              # :136-141
    add_fwd("rect_48x96", 48, 96, 0.37, 12, 90, [91, 92])
    add_fwd("rect_96x40", 96, 40, 0.6, 7, 93, [94])
    add_fwd("ties_64", 64, 64, 0.5, 8, 95, [96, 97], quantize_x=True)
    add_fwd("ragged_33x129", 33, 129, 0.41, 9, 98, [99])
    add_fwd("big_128x160", 128, 160, 0.3, 32, 100, [101, 102])
    g["fwd.names"] = np.array(fwd)

    # --- gather_matvec on random masks (test_layer.cpp:166-185) ------------------
    gm = []
    sel = R.uniform01(86, 20 * 40)
    for trial in range(6):
        rows, cols = 3 + trial * 5, 4 + trial * 6
        w = R.normal(870 + trial, rows * cols).reshape(rows, cols)
        x = R.normal(900 + trial, cols)
        kept = np.nonzero(sel[trial * 40: trial * 40 + cols] < 0.3)[0].astype(np.int64)
        y, touched = R.gather_matvec(w.T, x, kept, count_bytes=True)
        g[f"gmv.t{trial}.w"], g[f"gmv.t{trial}.x"] = w, x
        g[f"gmv.t{trial}.kept"], g[f"gmv.t{trial}.y"] = kept, y
        g[f"gmv.t{trial}.touched"] = np.array([touched], dtype=np.uint64)
        gm.append(f"t{trial}")
    g["gmv.names"] = np.array(gm)

    # --- io_cost KATs (test_layer.cpp:193-215) ------------------------------------
    io_cases = [(4096, 4096, 0.3, 1024), (4096, 4096, 0.5, 0), (4096, 4096, 1.0, 0),
                (96, 64, 0.37, 12), (4096, 11008, 0.5, 688), (11008, 4096, 0.5, 256)]
    io = []
    for (n, m, s, r) in io_cases:
        rep = R.io_cost(n, m, s, r)
        io.append([n, m, s, r, rep["dense_bytes"], rep["touched_bytes"], rep["relative_cost"]])
    g["io.cases"] = np.array(io, dtype=np.float64)

    # --- Recipe::plan_for (search.cpp:14-25) ----------------------------------------
    pf = []
    for (rho, c, n, m) in [(0.4, 0.5, 4096, 11008), (0.3, 0.5, 4096, 4096), (0.7, 0.5, 11008, 4096),
                           (0.0, 1.0, 64, 64), (1.0, 0.5, 64, 64), (0.5, 2.0, 10, 12),
                           (0.55, 0.5, 1024, 4096), (0.31, 0.5, 14336, 4096)]:
        s, r = R.plan_for(rho, c, n, m)
        pf.append([rho, c, n, m, s, r])
    g["plan.cases"] = np.array(pf, dtype=np.float64)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
