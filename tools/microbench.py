"""Per-linear timing of the fused kernel (CUDA events, L2-defeating rotation).

    python tools/microbench.py [--reps 50] [--copies 8] [--shapes q,gate,down]

For each shape, `copies` independent layers (> 2x L2 bytes in total) are
launched round-robin so every launch streams from HBM.  Reports the median
per-launch time, algorithmic GB/s and the fraction of MEASURED_PEAKS hbm_gbs,
for the R-Sparse forward and for the dense sweep of the same layer.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2504_19449_b200 as rsp  # noqa: E402
from paper_2504_19449_b200 import workloads as wl  # noqa: E402

SHAPES = {"q": (4096, 4096), "gate": (11008, 4096), "down": (4096, 11008), "kv3": (1024, 4096),
          "gate3": (14336, 4096), "down3": (4096, 14336)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--copies", type=int, default=8)
    ap.add_argument("--shapes", default="q,gate,down")
    ap.add_argument("--s", type=float, default=0.25)
    ap.add_argument("--rho", type=float, default=0.5, help="config-2 rho (overrides --s when > 0)")
    ap.add_argument("--wdt", default="bf16")
    ap.add_argument("--xdt", default="bf16")
    ap.add_argument("--graph", action="store_true", help="also time a graph of back-to-back launches")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    rng = np.random.default_rng(0)
    results = []
    for name in args.shapes.split(","):
        m, n = SHAPES[name]
        plan = rsp.Recipe([args.rho], [0.5]).plan_for(0, n, m) if args.rho > 0 else rsp.SparsityPlan(args.s, n // 16)
        layers, xs = [], []
        for c in range(args.copies):
            w = torch.randn(m, n, device=dev, dtype=torch.bfloat16) * 0.02
            a = torch.randn(m, plan.rank, device=dev, dtype=torch.bfloat16) * 0.05
            b = torch.randn(plan.rank, n, device=dev, dtype=torch.bfloat16) * 0.05
            layers.append(rsp.DecomposedLayer(w, a, b, plan, weight_dtype=args.wdt))
            x = torch.from_numpy(wl.heavy_tailed_x(n, rng)).to(dev)
            xs.append(x.to(torch.bfloat16) if args.xdt == "bf16" else x)
            del w, a, b
        y = torch.empty(m, device=dev)
        ws = layers[0].workspace()
        rep = layers[0].io_cost()
        info = layers[0].info

        def time_it(fn):
            for i in range(args.copies * 2):
                fn(i % args.copies)
            torch.cuda.synchronize()
            ts = []
            for i in range(args.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn(i % args.copies)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            return float(np.median(ts)), float(np.percentile(ts, 10))

        t_sp, t_sp10 = time_it(lambda i: layers[i].forward(xs[i], out=y, workspace=ws))
        t_de, t_de10 = time_it(lambda i: layers[i].dense_forward(xs[i], out=y, workspace=ws))
        r = {"shape": name, "m": m, "n": n, "k": info["k"], "r": plan.rank, "grid": info["grid"],
             "col_tiles": info["col_tiles"], "k_splits": info["k_splits"], "smem": info["smem_bytes"],
             "sparse_us": t_sp, "sparse_us_p10": t_sp10,
             "sparse_GBps": rep.kernel_total_bytes / t_sp / 1e3,
             "dense_us": t_de, "dense_GBps": rep.dense_weight_bytes / t_de / 1e3}
        r["sparse_frac"] = r["sparse_GBps"] / peak
        r["dense_frac"] = r["dense_GBps"] / peak
        if args.graph:
            ys = [torch.empty(m, device=dev) for _ in layers]
            st = rsp.Stack(layers, xs, ys)
            for _ in range(3):
                st.launch()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                st.launch()
            e1.record()
            e1.synchronize()
            r["graph_us_per_linear"] = e0.elapsed_time(e1) * 1e3 / (args.reps * len(layers))
            st.close()
        results.append(r)
        print(json.dumps(r), flush=True)
        for l in layers:
            l.close()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
