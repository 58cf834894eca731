"""Phase timeline of the fused kernel (rsp_debug_forward_trace).

Prints, per shape, the median / max over CTAs of each phase stamp in µs
since CTA start, and the spread of CTA start times.
"""
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

EV = {1: "after_griddep", 2: "x_loaded+hist", 3: "cut", 4: "lists", 10: "W_prefetch_issued",
      11: "stage1_rows", 12: "t_reds", 5: "stage1+arrive",
      6: "W_rows_done", 7: "barrier_waited", 8: "A_rows_done", 9: "end"}
SHAPES = {"q": (4096, 4096), "gate": (11008, 4096), "down": (4096, 11008)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="q,gate,down")
    ap.add_argument("--mhz", type=float, default=1965.0)
    ap.add_argument("--dense", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(0)
    for name in args.shapes.split(","):
        m, n = SHAPES[name]
        plan = rsp.Recipe([0.5], [0.5]).plan_for(0, n, m)
        layers = []
        for _ in range(4):
            w = torch.randn(m, n, device=dev, dtype=torch.bfloat16) * 0.02
            a = torch.randn(m, plan.rank, device=dev, dtype=torch.bfloat16) * 0.05
            b = torch.randn(plan.rank, n, device=dev, dtype=torch.bfloat16) * 0.05
            layers.append(rsp.DecomposedLayer(w, a, b, plan))
        x = torch.from_numpy(wl.heavy_tailed_x(n, rng)).to(dev).to(torch.bfloat16)
        y = torch.empty(m, device=dev)
        ws = layers[0].workspace()
        grid = layers[0].info["grid"]
        tr = torch.zeros(grid * 16, dtype=torch.int64, device=dev)
        for i in range(12):
            l = layers[i % 4]
            L.check(L.lib().rsp_debug_forward_trace(l.handle, x.data_ptr(), L.RSP_BF16, y.data_ptr(),
                                                    ws.data_ptr(), ws.numel(), tr.data_ptr(),
                                                    1 if args.dense else 0,
                                                    torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        t = tr.view(grid, 16).cpu().numpy()
        start = t[:, 0]
        print(f"== {name} m={m} n={n} k={layers[0].k} r={plan.rank} grid={grid} "
              f"tiles={layers[0].info['col_tiles']} dense={args.dense}")
        print(f"   CTA start spread (globaltimer): {(start.max() - start.min()) / 1e3:.2f} us")
        for ev, label in EV.items():
            col = t[:, ev] / args.mhz  # cycles -> us
            col = col[t[:, ev] > 0]
            if col.size:
                print(f"   {ev:2d} {label:22s} median {np.median(col):7.2f} us   max {col.max():7.2f} us")
        for l in layers:
            l.close()


if __name__ == "__main__":
    main()
