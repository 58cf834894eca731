"""Phase timeline of one batched forward (rsp_debug_set_batch_trace): medians and
maxima over the CTAs of the per-phase clock64 stamps, in us at --mhz."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2504_19449_b200 as rsp  # noqa: E402
from paper_2504_19449_b200 import _lib as L  # noqa: E402
from paper_2504_19449_b200 import workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mhz", type=float, default=1965.0)
a = ap.parse_args()
L.check(L.lib().rsp_debug_set_batch_trace(1), "trace on")
dev = torch.device("cuda:0")
rng = np.random.default_rng(3)
PH = ["cut", "stage-x", "lists", "stage1", "arrive", "Wrows", "tbar", "stage2", "combine"]
for name, m, n, s, r in [("q", 4096, 4096, 0.2, 610), ("gate", 11008, 4096, 0.27, 687), ("down", 4096, 11008, 0.19, 933)]:
    layer = rsp.DecomposedLayer(torch.randn(m, n, device=dev, dtype=torch.bfloat16) * 0.02,
                                torch.randn(m, r, device=dev, dtype=torch.bfloat16) * 0.05,
                                torch.randn(r, n, device=dev, dtype=torch.bfloat16) * 0.05,
                                rsp.SparsityPlan(s, r), weight_dtype="bf16")
    ws = layer.workspace()
    for B in [2, 16]:
        X = torch.from_numpy(np.stack([wl.heavy_tailed_x(n, rng) for _ in range(B)])).to(dev).to(torch.bfloat16)
        for _ in range(3):
            y = layer.forward(X, workspace=ws)
        torch.cuda.synchronize()
        buf = np.zeros(160 * 16, dtype=np.int64)
        L.check(L.lib().rsp_debug_batch_trace(buf.ctypes.data, 160), "trace")
        t = buf.reshape(160, 16)
        used = t[:, 8] > 0
        t = t[used] / a.mhz
        med = np.median(t, axis=0)
        mx = t.max(axis=0)
        print(f"{name} B={B} ctas={used.sum()}: " + " ".join(f"{PH[i]}={med[i]:.2f}/{mx[i]:.2f}" for i in range(0, 9)))
