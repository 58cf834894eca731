"""Config 3 (BASELINE.json configs[3]): the config-2 stack at batch B in
{1, 2, 4, 8, 16}, i.i.d. heavy-tailed tokens, each token with its own mask.

For every B, one step = all 224 linears of the stack over B tokens, captured
in one CUDA graph:
  * B >= 2: `rsp_linear_forward(batch=B)` per linear -- the union-of-masks
    tensor-core path (csrc/rsp_batch.cu), W rows of the union read once;
  * B == 1: the persistent stack kernel (bench.py's headline path) and, for
    reference, the per-linear launch of the same fused kernel;
  * dense: cuBLAS bf16 GEMM [m, n] x [n, B] per layer group (fused QKV,
    gate/up), graph-captured.
Prints one JSON line per B (us/token = step time / B).

    python tools/batch_bench.py [--layers 32] [--steps 10] [--warmup 3] [--batches 1,2,4,8,16]
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


def time_graph(fn, steps, warmup, stream):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / steps  # ms per step


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batches", default="1,2,4,8,16")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    plans = wl.config2_plans(n_layers=a.layers)
    gid, wait = wl.input_groups(plans)
    gen = torch.Generator(device=dev)
    gen.manual_seed(4321)
    layers = []
    for (name, m, n, s, r) in plans:
        w = torch.randn(m, n, device=dev, dtype=torch.bfloat16, generator=gen) * 0.02
        am = torch.randn(m, r, device=dev, dtype=torch.bfloat16, generator=gen) * 0.05
        bm = torch.randn(r, n, device=dev, dtype=torch.bfloat16, generator=gen) * 0.05
        layers.append(rsp.DecomposedLayer(w, am, bm, rsp.SparsityPlan(s, r), weight_dtype="bf16"))
        del w, am, bm
    stream = torch.cuda.Stream()
    rng = np.random.default_rng(7)
    ngroups = max(gid) + 1
    gfirst = [gid.index(g) for g in range(ngroups)]
    # dense weights per input group (fused QKV / gate-up), for cuBLAS
    dgen = torch.Generator(device=dev)
    dgen.manual_seed(9)
    dense_w = []
    for g in range(ngroups):
        idx = [i for i in range(len(plans)) if gid[i] == g]
        dense_w.append(torch.randn(sum(plans[i][1] for i in idx), plans[idx[0]][2], device=dev,
                                   dtype=torch.bfloat16, generator=dgen) * 0.02)
    for B in [int(b) for b in a.batches.split(",")]:
        xs = []
        for g in range(ngroups):
            n = plans[gfirst[g]][2]
            name = plans[gfirst[g]][0]
            X = np.stack([wl.silu_gate_x(n, rng) if name.endswith("down_proj") else wl.heavy_tailed_x(n, rng)
                          for _ in range(B)])
            xs.append(torch.from_numpy(X).to(dev).to(torch.bfloat16))
        ys = [torch.empty((B, l.m_out), device=dev, dtype=torch.float32) for l in layers]
        wss = [l.workspace() for l in layers]
        res = {"config": "config3", "batch": B, "layers": a.layers, "linears": len(layers), "dtype": "bf16"}
        with torch.cuda.stream(stream):
            if B == 1:
                st = rsp.Stack(layers, [xs[gid[i]][0] for i in range(len(layers))],
                               [ys[i][0] for i in range(len(layers))], wait_prev=wait)
                ms = time_graph(lambda: st.launch(stream), a.steps, a.warmup, stream)
                res["stack_us_per_token"] = ms * 1e3
                st.close()
            if 1 < B <= 8:
                # B independent per-token persistent stacks on disjoint SM partitions
                tp = rsp.TokenParallelStack(layers, [xs[gid[i]] for i in range(len(layers))], ys, wait_prev=wait,
                                            stream=stream)
                ms = time_graph(lambda: tp.launch(stream), a.steps, a.warmup, stream)
                res["token_parallel_us_per_token"] = ms * 1e3 / B
                res["token_parallel_graph"] = tp.graph is not None
                tp.close()

            def step():
                for i, l in enumerate(layers):
                    l.forward(xs[gid[i]] if B > 1 else xs[gid[i]][0], out=ys[i] if B > 1 else ys[i][0],
                              workspace=wss[i], stream=stream)
            step()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step()
            ms = time_graph(lambda: g.replay(), a.steps, a.warmup, stream)
            res["per_linear_us_per_token"] = ms * 1e3 / B
            del g
            outs = [torch.empty((B, W.shape[0]), device=dev, dtype=torch.bfloat16) for W in dense_w]

            def dense():
                for gi, W in enumerate(dense_w):
                    torch.matmul(xs[gi], W.t(), out=outs[gi])
            dense()
            torch.cuda.synchronize()
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g2, stream=stream):
                dense()
            ms = time_graph(lambda: g2.replay(), a.steps, a.warmup, stream)
            res["dense_cublas_us_per_token"] = ms * 1e3 / B
            del g2
        best = min(v for k, v in res.items()
                   if k in ("stack_us_per_token", "per_linear_us_per_token", "token_parallel_us_per_token"))
        res["speedup_vs_dense_cublas"] = res["dense_cublas_us_per_token"] / best
        print(json.dumps(res), flush=True)
        del ys, xs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
