"""Time the stand-alone one-CTA selector (rsp_top_k_by_magnitude)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_19449_b200 as rsp  # noqa: E402
from paper_2504_19449_b200 import workloads as wl  # noqa: E402

rng = np.random.default_rng(0)
for n in (4096, 11008):
    for dt in (torch.float32, torch.bfloat16):
        x = torch.from_numpy(wl.heavy_tailed_x(n, rng)).cuda().to(dt)
        k = n // 4
        for _ in range(10):
            rsp.top_k_by_magnitude(x, k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            rsp.top_k_by_magnitude(x, k)
        e1.record()
        e1.synchronize()
        print(f"select n={n} {dt}: {e0.elapsed_time(e1) / 200 * 1e3:.2f} us/launch")
