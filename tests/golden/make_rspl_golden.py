"""Generate tests/golden/rspl/*.rspl and rspl.npz with the REFERENCE library.

    python tests/golden/make_rspl_golden.py     (needs oracle/_ref)

Valid files come from rsparse::write_decomposed_layer (layer.cpp:243-267) on
reference-decomposed layers; the expected contents and forward outputs come
from rsparse::read_decomposed_layer (layer.cpp:269-301) and rsparse::forward
on the layer read back.  Malformed files are byte edits of a valid one, each
named for the io_error the reference raises on it (checked here against the
reference reader itself).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import OracleError, ref_oracle  # noqa: E402

OUT_DIR = os.path.join(HERE, "rspl")
OUT_NPZ = os.path.join(HERE, "rspl.npz")


def main():
    R = ref_oracle()
    os.makedirs(OUT_DIR, exist_ok=True)
    g = {}
    names = []
    for (name, m, n, s, r, wseed, xseeds) in [
        ("l48x96", 48, 96, 0.37, 12, 90, [91, 92]),
        ("l64x64_r0", 64, 64, 0.5, 0, 120, [121]),
        ("l20x24_s0", 20, 24, 0.0, 5, 75, [77]),
    ]:
        w = R.normal(wseed, m * n).reshape(m, n)
        a, b, comps = R.decompose_uniform(w, s, r)
        comps = comps[::-1].copy()  # non-trivial component ids exercise the field
        path = os.path.join(OUT_DIR, f"{name}.rspl")
        R.write_layer(path, w.T, a, b, s, comps)
        d = R.read_layer(path)
        g[f"{name}.w_cols"], g[f"{name}.a_r"], g[f"{name}.b_r"] = d["w_cols"], d["a_r"], d["b_r"]
        g[f"{name}.comps"] = d["comps"]
        g[f"{name}.plan"] = np.array([d["keep_fraction"], d["rank"]], dtype=np.float64)
        xs = np.stack([R.normal(sd, n) for sd in xseeds])
        g[f"{name}.x"] = xs
        g[f"{name}.y"] = np.stack([R.forward(d["w_cols"], d["a_r"], d["b_r"], d["keep_fraction"], x)
                                  for x in xs])
        names.append(name)
    g["names"] = np.array(names)

    src = open(os.path.join(OUT_DIR, "l48x96.rspl"), "rb").read()
    bad = {
        "bad_magic": b"RSPX" + src[4:],
        "bad_version": src[:4] + bytes([2]) + src[5:],
        "truncated_header": src[:11],
        "truncated_body": src[: len(src) // 2],
        "truncated_plan": src[:-4],
        "bad_rank_field": src[:-8] + np.array([13.0]).tobytes(),
    }
    for name, data in bad.items():
        path = os.path.join(OUT_DIR, f"{name}.rspl")
        with open(path, "wb") as f:
            f.write(data)
        try:
            R.read_layer(path)
        except OracleError as e:
            assert e.status == 3, (name, e.status)  # io_error
        else:
            raise AssertionError(f"reference accepted {name}")
    g["bad_names"] = np.array(sorted(bad))
    np.savez_compressed(OUT_NPZ, **g)
    print(f"wrote {OUT_NPZ} and {len(names) + len(bad)} files under {OUT_DIR}")


if __name__ == "__main__":
    main()
