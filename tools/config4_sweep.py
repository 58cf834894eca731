"""Config 4 (BASELINE.json configs[4]): Llama-3-8B-shaped 32-layer stack, bf16,
batch 1, model-level sparsity in {30..70}% x rank in {64, 128, 256, 512}
(workloads.config4_plans; infeasible k/v plans clamped and reported), 16
outlier channels in the heavy-tailed inputs.  Each point: the persistent
stack kernel (bench.py's path), CUDA events, no flush needed (> 14 GB of
operands).  One JSON line per point, then the dense cuBLAS stack (fused
QKV / gate-up) once for reference.

    python tools/config4_sweep.py [--layers 32] [--steps 10] [--warmup 3]
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


def timed(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--sparsities", default="0.3,0.4,0.5,0.6,0.7")
    ap.add_argument("--ranks", default="64,128,256,512")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6550.0) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6550.0
    gen = torch.Generator(device=dev)
    gen.manual_seed(11)
    shapes = {}
    for (name, m, n) in wl.LLAMA3_8B:  # one random W per shape, shared by the layers of the stack
        shapes[name] = torch.randn(m, n, device=dev, dtype=torch.bfloat16, generator=gen) * 0.02
    rng = np.random.default_rng(4)
    for sp in [float(v) for v in a.sparsities.split(",")]:
        for rank in [int(v) for v in a.ranks.split(",")]:
            plans, clamped = wl.config4_plans(sp, rank, a.layers)
            gid, wait = wl.input_groups(plans)
            layers, xs = [], {}
            for i, (name, m, n, s, r) in enumerate(plans):
                short = name.rsplit(".", 1)[1]
                am = torch.randn(m, r, device=dev, dtype=torch.bfloat16, generator=gen) * 0.05
                bm = torch.randn(r, n, device=dev, dtype=torch.bfloat16, generator=gen) * 0.05
                layers.append(rsp.DecomposedLayer(shapes[short], am, bm, rsp.SparsityPlan(s, r), weight_dtype="bf16"))
                del am, bm
                if gid[i] not in xs:
                    x = wl.silu_gate_x(n, rng) if short == "down_proj" else wl.heavy_tailed_x(n, rng, outliers=16)
                    xs[gid[i]] = torch.from_numpy(x).to(dev).to(torch.bfloat16)
            ys = [torch.empty(l.m_out, device=dev) for l in layers]
            st = rsp.Stack(layers, [xs[gid[i]] for i in range(len(layers))], ys, wait_prev=wait)
            ms = timed(lambda: st.launch(), a.steps, a.warmup)
            import importlib.util as _iu
            _spec = _iu.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
            _bm = _iu.module_from_spec(_spec)
            _spec.loader.exec_module(_bm)
            alg = _bm.algorithmic_bytes(layers)  # SURVEY 8(d) model (S^c rows of b_r)
            ref = sum(l.io_cost().touched_bytes for l in layers)
            dense = sum(2 * m * n for (_, m, n, _, _) in plans)
            res = {"config": "config4", "sparsity": sp, "rank": rank, "layers": a.layers, "us_per_token": ms * 1e3,
                   "algorithmic_GB": alg / 1e9, "achieved_GBps": alg / (ms * 1e-3) / 1e9,
                   "roofline_frac": alg / (ms * 1e-3) / 1e9 / peak, "kernel_bytes_vs_dense": alg / dense,
                   "clamped": [{"linear": c[0], "rank": c[1], "clamped_to": c[2]} for c in clamped]}
            print(json.dumps(res), flush=True)
            st.close()
            del layers, ys, st
            torch.cuda.empty_cache()
    # dense cuBLAS stack for reference (fused QKV / gate-up)
    groups = [("attn", ["q_proj", "k_proj", "v_proj"]), ("o", ["o_proj"]), ("mlp", ["gate_proj", "up_proj"]),
              ("down", ["down_proj"])]
    ws = [torch.cat([shapes[nm] for nm in names], 0) for _, names in groups]
    xv = [torch.randn(w.shape[1], device=dev, dtype=torch.bfloat16) for w in ws]
    outs = [torch.empty(w.shape[0], device=dev, dtype=torch.bfloat16) for w in ws]

    def dense_step():
        for _ in range(a.layers):
            for w, x, o in zip(ws, xv, outs):
                torch.matmul(w, x, out=o)
    dense_step()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        dense_step()
    ms = timed(lambda: g.replay(), a.steps, a.warmup)
    print(json.dumps({"config": "config4", "dense_cublas_us_per_token": ms * 1e3,
                      "note": "same W per layer (L2 cannot hold it: 436 MB per layer)"}), flush=True)


if __name__ == "__main__":
    main()
