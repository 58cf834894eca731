#!/usr/bin/env python
"""Benchmark: µs/token of the config-2 R-Sparse linear stack (BASELINE.json).

Workload (BASELINE.json configs[2]): the 224 linears of a 32-layer
Llama-2-7B-shaped stack (q/k/v/o 4096x4096, gate/up 11008x4096, down
4096x11008), bf16 weights, bf16 activations, fp32 accumulation, batch 1,
per-linear (s, r) from Recipe::plan_for with rho ~ U(0.3, 0.7), C = 0.5
(50% model-level sparsity by the reference io_cost).  Synthetic random-init
weights (no checkpoints offline); heavy-tailed synthetic activations
(Laplace x LogNormal, 8 outliers x20; SiLU(g)*u for down_proj).

One step = one decode token through all 224 linears in decode order: ONE
persistent stack-kernel launch (CUDA graph) with a grid barrier wherever a
linear's input is the previous output; q/k/v (and gate/up), which read the
same activation in a Llama decoder layer, run side by side on disjoint CTA
partitions (workloads.input_groups).  The resident operands (~16 GB) dwarf
the 126 MB L2, so no flush is needed between steps.  N > 1: every linear is
row-sharded over the ranks and followed by one NCCL all-gather of y
(SURVEY §8(e)).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "µs/token per R-Sparse linear stack & touched-bytes HBM GB/s vs dense GEMV"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=32, help="decoder layers in the stack")
    ap.add_argument("--no-dense", action="store_true", help="skip the dense baselines")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no extras)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="use the row-sharded + all-gather path even on one rank (exercises it on 1 GPU)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.out = ""

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.out = ""

    def summary(self):
        rows = []
        for line in self.out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[4:8]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for (_, _, flags) in rows for i, f in enumerate(flags)
                          if f.lower() == "active"})
        sm = [r[0] for r in rows]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------------------- workload
def build_stack(rsp, wl, plans, rank, world, dev, torch):
    """Create every linear's shard on the device from synthetic weights, and
    one synthetic activation per input group (q/k/v share one, gate/up share
    one: workloads.input_groups)."""
    rng = np.random.default_rng(1234)
    gen = torch.Generator(device=dev)
    gen.manual_seed(4321)
    gid, wait = wl.input_groups(plans)
    layers, xs_host = [], []
    for i, (name, m, n, s, r) in enumerate(plans):
        w = torch.randn(m, n, device=dev, dtype=torch.bfloat16, generator=gen) * 0.02
        a = torch.randn(m, r, device=dev, dtype=torch.bfloat16, generator=gen) * 0.05
        b = torch.randn(r, n, device=dev, dtype=torch.bfloat16, generator=gen) * 0.05
        layers.append(rsp.DecomposedLayer(w, a, b, rsp.SparsityPlan(s, r), weight_dtype="bf16",
                                          device=dev.index, shard_rank=rank, shard_count=world))
        del w, a, b
        if wait[i]:
            xs_host.append(wl.silu_gate_x(n, rng) if name.endswith("down_proj") else wl.heavy_tailed_x(n, rng))
    torch.cuda.synchronize()
    return layers, xs_host, gid, wait


def kernel_bytes(layers):
    """Algorithmic bytes per step (SURVEY §8(d) model, this rank's shards):
    elem*(k*m + (n-k)*r + r*m) + x + y, summed over the stack."""
    tot = 0
    for l in layers:
        rep = l.io_cost()
        tot += rep.kernel_total_bytes
    return tot


def time_graph(torch, launch, steps, warmup, stream, barrier=None):
    for _ in range(warmup):
        launch()
    torch.cuda.synchronize()
    if barrier:
        barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(stream)
    for (a, b) in evs:
        a.record(stream)
        launch()
        b.record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    if barrier:
        barrier()
    per = [a.elapsed_time(b) for (a, b) in evs]
    return t0.elapsed_time(t1), per


def cpu_reference_leg(wl, plans, threads, seconds=None, warmup=1, passes=None):
    """The reference's own CPU forward (oracle/_ref = reference sources compiled
    in place; else the C port) over one decoder layer's 7 linears per pass,
    linears spread over `threads` host threads; extrapolated to the stack."""
    from oracle.oracle import c_oracle, ref_available, ref_oracle
    sample = plans[:7]
    rng = np.random.default_rng(99)
    use_ref = ref_available()
    R = ref_oracle() if use_ref else c_oracle()
    objs, xs, ys = [], [], []
    for (name, m, n, s, r) in sample:
        w_cols = rng.standard_normal((n, m)) * 0.02
        a = rng.standard_normal((m, r)) * 0.05
        b = rng.standard_normal((r, n)) * 0.05
        x = (wl.silu_gate_x(n, rng) if name.endswith("down_proj") else wl.heavy_tailed_x(n, rng)).astype(np.float64)
        objs.append(R.layer(w_cols, a, b, s) if use_ref else (w_cols, a, b, s))
        xs.append(x)
        ys.append(np.empty(m))

    def one_pass():
        if use_ref:
            R.forward_many(objs, xs, ys, threads)
        else:
            R.forward_many(objs, xs, threads)

    for _ in range(max(warmup, 0)):
        one_pass()
    times = []
    t_end = time.perf_counter() + (seconds or 0.0)
    while (passes is not None and len(times) < passes) or \
            (passes is None and (time.perf_counter() < t_end or len(times) < 3)):
        t = time.perf_counter()
        one_pass()
        times.append(time.perf_counter() - t)
    layer_s = float(np.median(times))
    scale = len(plans) / len(sample)
    return {
        "value": layer_s * 1e6 * scale, "unit": "us/token", "cores": threads,
        "kind": "reference" if use_ref else "port",
        "sample": (f"{'reference rsparse::forward (oracle/_ref, fp64, -O3)' if use_ref else 'C port'} over "
                   f"decoder layer 0's 7 linears of the config-2 stack per pass, linears spread over "
                   f"{threads} threads, median of {len(times)} passes, x{scale:g} to the {len(plans)}-linear stack"),
        "passes": len(times), "pass_times_s": times,
    }


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2504_19449_b200 import workloads as wl
    plans = wl.config2_plans(n_layers=args.layers)
    threads = os.cpu_count() or 1
    res = cpu_reference_leg(wl, plans, threads, warmup=args.warmup, passes=args.steps)
    line = {
        "metric": METRIC, "impl": "reference", "value": res["value"], "unit": "us/token",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": res["value"] / 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config2: 32-layer Llama-2-7B-shaped R-Sparse linear stack, batch 1, "
                               "50% model-level sparsity (rho~U(0.3,0.7), C=0.5)",
                   "global_batch": 1, "layers": args.layers, "linears": len(plans)},
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": res["value"], "unit": "us/token", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1 or args.force_sharded:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
    import paper_2504_19449_b200 as rsp
    from paper_2504_19449_b200 import workloads as wl
    rsp.lib()

    plans = wl.config2_plans(n_layers=args.layers)
    layers, xs_host, gid, wait = build_stack(rsp, wl, plans, rank, world, dev, torch)

    # activations: one contiguous bf16 buffer (device + pinned host) for the e2e copy
    offs = np.cumsum([0] + [x.size for x in xs_host])
    x_host = torch.empty(int(offs[-1]), dtype=torch.bfloat16).pin_memory()
    x_host.copy_(torch.from_numpy(np.concatenate(xs_host)).to(torch.bfloat16))
    x_dev = x_host.to(dev)
    xg = [x_dev[offs[g]:offs[g + 1]] for g in range(len(xs_host))]
    xs = [xg[gid[i]] for i in range(len(layers))]
    mloc = [l.row_end - l.row_begin for l in layers]
    mfull = [l.m_out for l in layers]
    yoffs = np.cumsum([0] + (mfull if world > 1 else mloc))
    y_dev = torch.empty(int(yoffs[-1]), dtype=torch.float32, device=dev)
    y_host = torch.empty_like(y_dev, device="cpu").pin_memory()
    ys = [y_dev[yoffs[i]:yoffs[i + 1]] for i in range(len(layers))]
    stream = torch.cuda.Stream(device=dev)

    sharded = world > 1 or args.force_sharded
    if not sharded:
        # one persistent launch per token; q/k/v and gate/up overlap (shared input)
        st = rsp.Stack(layers, xs, ys, wait_prev=wait)
        launch = lambda: st.launch(stream)  # noqa: E731
    else:
        # row-sharded linears, each followed by one in-place NCCL all-gather
        # of y (paper_2504_19449_b200/sharding.py), captured as one graph
        from paper_2504_19449_b200.sharding import ShardedGroupStack, ShardedStack, even_shards
        if all(even_shards(l.m_out, world) for l in layers) and not os.environ.get("RSP_PER_LINEAR_SHARDS"):
            st = ShardedGroupStack(layers, xs, ys, gid, stream=stream)  # one stack launch per input group
        else:
            st = ShardedStack(layers, xs, ys, stream=stream)
        launch = st.launch

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    with torch.cuda.stream(stream):
        with ClockSampler(local) as clocks:
            total_ms, per = time_graph(torch, launch, args.steps, args.warmup, stream, barrier)
    ms_step = total_ms / args.steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms_step], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    us_token = ms_step * 1e3

    bytes_step = kernel_bytes(layers)  # this rank's algorithmic bytes
    hbm_peak, peak_kind = measured_peaks()
    achieved = bytes_step / (ms_step * 1e-3) / 1e9

    # ---- end to end: H2D of the token's activations, the stack, D2H of all outputs ----
    h2d = x_host.numel() * 2
    d2h = y_dev.numel() * 4

    def e2e_step():
        x_dev.copy_(x_host, non_blocking=True)
        launch()
        y_host.copy_(y_dev, non_blocking=True)

    with torch.cuda.stream(stream):
        e2e_total, _ = time_graph(torch, e2e_step, args.steps, args.warmup, stream, barrier)
    e2e_ms = e2e_total / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    extras = {}
    if not args.no_dense and not args.profile and world == 1:
        extras.update(dense_baselines(torch, rsp, layers, xs, ys, stream, args, plans, dev, gid, wait))

    out = {
        "metric": METRIC, "value": us_token, "unit": "us/token", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": False, "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "config2: 32-layer Llama-2-7B-shaped R-Sparse linear stack, batch 1, "
                               "50% model-level sparsity (rho~U(0.3,0.7), C=0.5), bf16 W/x, fp32 accum; "
                               "q/k/v and gate/up share one input (decoder-layer dataflow)",
                   "global_batch": 1, "layers": args.layers, "linears": len(layers),
                   "parallelism": f"row-shard{world}" + ("+allgather" if sharded else ""),
                   "sharded_graph": (getattr(st, "graph", None) is not None) if sharded else None,
                   "l2": "no flush: 16 GB resident operands >> 126 MB L2",
                   "step_ms_p10_p50_p90": [float(np.percentile(per, q)) for q in (10, 50, 90)]},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": None if sharded else load_traffic(),
                     "peak_kind": peak_kind, "algorithmic_bytes_per_step": bytes_step,
                     "kernel": ("stack_kernel<bf16,bf16> (1 launch per input group, + NCCL all-gather of y)" if sharded
                                else "stack_kernel<bf16,bf16> (1 persistent launch/step, 224 linears)")},
        "e2e": {"value": e2e_ms * 1e3, "unit": "us/token", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": args.steps * (max(gid) + 1 if sharded else 1),
        "clocks": clocks.summary(),
    }
    out.update(extras)
    if "dense_cublas_us_per_token" in out:
        out["speedup_vs_dense_cublas"] = out["dense_cublas_us_per_token"] / us_token
        out["speedup_vs_dense_inhouse"] = out["dense_inhouse_us_per_token"] / us_token
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        out["cpu_baseline"] = {k: v for k, v in cpu_reference_leg(wl, plans, os.cpu_count() or 1,
                                                                  seconds=args.cpu_seconds).items()
                               if k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if sharded:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


def load_traffic():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_launch")
    return None


def dense_baselines(torch, rsp, layers, xs, ys, stream, args, plans, dev, gid, wait):
    """Dense bf16 GEMV stacks of the same layers under the same protocol:
    (1) the in-house kernel over all m_in channels (same persistent stack,
    same overlap of shared-input linears), (2) cuBLAS (torch.matmul on
    row-major bf16 W, graph-captured) with the shared-input linears of a layer
    concatenated into one GEMV (fused QKV and gate/up, as production decode
    does), which is the strongest dense baseline."""
    res = {}
    st = rsp.Stack(layers, xs, ys, dense=True, wait_prev=wait)
    with torch.cuda.stream(stream):
        tot, _ = time_graph(torch, lambda: st.launch(stream), args.steps, args.warmup, stream)
    res["dense_inhouse_us_per_token"] = tot / args.steps * 1e3
    st.close()
    gen = torch.Generator(device=dev)
    gen.manual_seed(7)
    groups = []
    for g in range(max(gid) + 1):
        idx = [i for i in range(len(plans)) if gid[i] == g]
        m = sum(plans[i][1] for i in idx)
        n = plans[idx[0]][2]
        groups.append((torch.randn(m, n, device=dev, dtype=torch.bfloat16, generator=gen) * 0.02,
                       xs[idx[0]], torch.empty(m, device=dev, dtype=torch.bfloat16)))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        for W, x, o in groups:
            torch.matmul(W, x, out=o)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=stream):
            for W, x, o in groups:
                torch.matmul(W, x, out=o)
        tot, _ = time_graph(torch, lambda: g.replay(), args.steps, args.warmup, stream)
    res["dense_cublas_us_per_token"] = tot / args.steps * 1e3
    dense_bytes = sum(2 * m * n for (_, m, n, _, _) in plans)
    res["dense_cublas_GBps"] = dense_bytes / (tot / args.steps * 1e-3) / 1e9
    del groups, g
    torch.cuda.empty_cache()
    return res


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    res = run_ours(args)
    return res


if __name__ == "__main__":
    sys.exit(main())
