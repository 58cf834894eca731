"""Time one batched linear forward (config-1 shapes, bf16) per batch size:
CUDA events around rsp_linear_forward(batch=B), plus the batch-1 forward."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2504_19449_b200 as rsp  # noqa: E402
from paper_2504_19449_b200 import workloads as wl  # noqa: E402

dev = torch.device("cuda:0")
rng = np.random.default_rng(3)
SHAPES = [("q", 4096, 4096, 0.2, 610), ("gate", 11008, 4096, 0.27, 687), ("down", 4096, 11008, 0.19, 933)]
ONLY = os.environ.get("BATCH_PROBE")  # e.g. "q:16" for a profiler run
for name, m, n, s, r in SHAPES:
    if ONLY and name != ONLY.split(":")[0]:
        continue
    w = torch.randn(m, n, device=dev, dtype=torch.bfloat16) * 0.02
    a = torch.randn(m, r, device=dev, dtype=torch.bfloat16) * 0.05
    b = torch.randn(r, n, device=dev, dtype=torch.bfloat16) * 0.05
    layer = rsp.DecomposedLayer(w, a, b, rsp.SparsityPlan(s, r), weight_dtype="bf16")
    ws = layer.workspace()
    for B in ([int(ONLY.split(':')[1])] if ONLY else [1, 2, 4, 8, 16]):
        X = torch.from_numpy(np.stack([wl.heavy_tailed_x(n, rng) for _ in range(B)])).to(dev).to(torch.bfloat16)
        x = X if B > 1 else X[0]
        out = torch.empty((B, m) if B > 1 else (m,), device=dev)
        for _ in range(3):
            layer.forward(x, out=out, workspace=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            layer.forward(x, out=out, workspace=ws)
        e1.record()
        e1.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        print(f"{name:5s} B={B:2d}: {us:8.1f} us per forward ({us / B:7.1f} us/token)", flush=True)
