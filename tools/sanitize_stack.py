"""A small config-2-like stack (one decoder layer at reduced width, grouped
q/k/v and gate/up, bf16) plus single and batched forwards, launched a few
times: a workload for compute-sanitizer memcheck / racecheck / synccheck
where the sanitizer is allowed (it is closed on this project's GPU pool, where
the bounds-checked build, tools/gpu_debugchecks.sh, runs instead).  Exits
non-zero on a parity failure."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2504_19449_b200 as rsp  # noqa: E402
from paper_2504_19449_b200 import workloads as wl  # noqa: E402
from oracle.oracle import c_oracle  # noqa: E402  (checker only)


def main():
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(0)
    shapes = [("q_proj", 512, 512), ("k_proj", 512, 512), ("v_proj", 512, 512), ("o_proj", 512, 512),
              ("gate_proj", 1376, 512), ("up_proj", 1376, 512), ("down_proj", 512, 1376)]
    plans = [(f"layers.0.{n}", m, k, 0.25, 64 if i % 2 else 120) for i, (n, m, k) in enumerate(shapes)]
    gid, wait = wl.input_groups(plans)
    layers, xs, xg = [], [], {}
    for i, (name, m, n, s, r) in enumerate(plans):
        w = torch.randn(m, n, device=dev) * 0.02
        a = torch.randn(m, r, device=dev) * 0.05
        b = torch.randn(r, n, device=dev) * 0.05
        layers.append(rsp.DecomposedLayer(w, a, b, rsp.SparsityPlan(s, r), weight_dtype="bf16"))
        if gid[i] not in xg:
            xg[gid[i]] = torch.from_numpy(wl.heavy_tailed_x(n, rng)).to(dev).to(torch.bfloat16)
        xs.append(xg[gid[i]])
    ys = [torch.empty(l.m_out, device=dev) for l in layers]
    st = rsp.Stack(layers, xs, ys, wait_prev=wait)
    for _ in range(2):
        st.launch()
    torch.cuda.synchronize()
    C = c_oracle()
    bad = 0
    for l, x, y, p in zip(layers, xs, ys, plans):
        W, A, B = l.export()
        yo = C.forward(np.ascontiguousarray(W.T), A, B, p[3], x.float().cpu().numpy().astype(np.float64))
        e = np.max(np.abs(y.cpu().numpy() - yo)) / np.max(np.abs(yo))
        bad += e > 1e-5
    # single-linear forward and the batched (B = 4) path on the same layers
    X = torch.stack([torch.from_numpy(wl.heavy_tailed_x(512, rng)) for _ in range(4)]).to(dev).to(torch.bfloat16)
    for l in layers[:4]:
        l.forward(X[0])
        l.forward(X)
    torch.cuda.synchronize()
    print("sanitize workload done, parity failures:", bad)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
