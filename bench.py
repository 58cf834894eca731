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
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "µs/token per R-Sparse linear stack & touched-bytes HBM GB/s vs dense GEMV"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=32, help="decoder layers in the stack")
    ap.add_argument("--no-dense", action="store_true", help="skip the dense baselines")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--cpu-layers", type=int, default=4,
                    help="decoder layers in the cpu_baseline sample of the GPU arm (one token through them)")
    ap.add_argument("--ref-layers", type=int, default=None,
                    help="--impl reference: decoder layers per pass, scaled to --layers (default: all of them, "
                         "or a bounded sample when --steps would take more than ~4 minutes)")
    ap.add_argument("--deterministic", action="store_true",
                    help="fixed-order (bit-reproducible) combines instead of float reductions at L2")
    ap.add_argument("--check", action="store_true",
                    help="after the timed loop, check a sample of the stack outputs against the oracle")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no extras)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "kernel"],
                    help="row-sharded runs: y assembled by NCCL all-gathers after each group's launch, or by "
                         "the kernel's own stores into every rank's y over peer memory (PeerStack)")
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
def build_stack(rsp, wl, plans, rank, world, dev, torch, deterministic=False):
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
                                          device=dev.index, shard_rank=rank, shard_count=world,
                                          deterministic=deterministic))
        del w, a, b
        if wait[i]:
            xs_host.append(wl.silu_gate_x(n, rng) if name.endswith("down_proj") else wl.heavy_tailed_x(n, rng))
    torch.cuda.synchronize()
    return layers, xs_host, gid, wait


def algorithmic_bytes(layers):
    """Algorithmic bytes per step (SURVEY §8(d) model, this rank's shards):
    elem*(k*m + (n-k)*r + r*m) + x + y with padded widths, summed over the
    stack -- the S^c rows of b_r only, whatever the kernel actually reads."""
    tot = 0
    for l in layers:
        info = l.info
        m, n, k, r = info["m_pad"], info["m_in"], info["k"], info["rank"]
        rp = info["r_pad"]
        lr = r > 0 and k < n
        tot += 2 * (k * m + ((n - k) * rp + r * m if lr else 0)) + 4 * n + 4 * (info["row_end"] - info["row_begin"])
    return tot


def kernel_bytes(layers):
    """Bytes the kernels read per step (rsp_linear_io_cost: the residual form
    of bf16 layers reads every row of b_r^T, n r instead of (n - k) r)."""
    return sum(l.io_cost().kernel_total_bytes for l in layers)


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


# --------------------------------------------------------------------------- reference CPU arm
# The reference arm never imports paper_2504_19449_b200 (nor maps its .so):
# plans come from the reference's own Recipe::plan_for (oracle/_ref), the
# draws replicate workloads.config2_plans (same numpy generator and order).
REF_SHAPES = [("q_proj", 4096, 4096), ("k_proj", 4096, 4096), ("v_proj", 4096, 4096),
              ("o_proj", 4096, 4096), ("gate_proj", 11008, 4096), ("up_proj", 11008, 4096),
              ("down_proj", 4096, 11008)]
REF_GROUP = {"q_proj": 0, "k_proj": 0, "v_proj": 0, "o_proj": 1, "gate_proj": 2, "up_proj": 2, "down_proj": 3}


def ref_config2_plans(R, n_layers=32, seed=2, budget=0.5):
    """(name, m_out, m_in, s, r) per linear: rho ~ U(0.3, 0.7), C = 0.5 through
    the reference's Recipe::plan_for (search.cpp:14-25) -- the same draws as
    workloads.config2_plans (checked by tests/test_bench_cpu.py)."""
    rng = np.random.default_rng(seed)
    out = []
    for layer in range(n_layers):
        for (name, m, n) in REF_SHAPES:
            rho = float(rng.uniform(0.3, 0.7))
            s, r = R.plan_for(rho, budget, n, m)
            out.append((f"layers.{layer}.{name}", m, n, float(s), int(r)))
    return out


def host_info():
    info = {"nproc": os.cpu_count()}
    try:
        info["affinity"] = len(os.sched_getaffinity(0))
    except Exception:
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith(("MemTotal", "MemAvailable")):
                    info[line.split(":")[0]] = int(line.split()[1]) * 1024
    except Exception:
        pass
    return info


def cpu_reference_leg(plans, threads, seconds=None, warmup=1, passes=None, layers=None):
    """The reference's own CPU forward (oracle/_ref = the reference sources
    compiled in place; else the C port) over the config-2 stack.

    A pass is one decode token through ``layers`` decoder layers (default:
    all of them).  Layers are built one at a time (fp64 weights of one layer
    resident: ~2 GB), and every layer's 7 linears are run in decode order:
    the linears of one input group (q/k/v, o, gate/up, down) concurrently on
    up to ``threads`` host threads (rsparse::forward is single-threaded and
    re-entrant), groups one after another.  Only the forward
    calls are timed; each pass's time is the sum over its layers, so the
    reported per-token time covers exactly the work that ran."""
    from oracle.oracle import c_oracle, ref_available, ref_oracle
    use_ref = ref_available()
    R = ref_oracle() if use_ref else c_oracle()
    rng = np.random.default_rng(99)
    n_layers = len(plans) // 7 if layers is None else layers
    rmax = max(p[4] for p in plans[: 7 * n_layers])
    src = {}
    for (name, m, n) in REF_SHAPES:  # fp64 sources per shape (values do not change the work)
        if (m, n) not in src:
            src[(m, n)] = (rng.standard_normal((n, m)) * 0.02, rng.standard_normal((m, rmax)) * 0.05,
                           rng.standard_normal((rmax, n)) * 0.05)
    xs = {}
    for (name, m, n) in REF_SHAPES:
        g = REF_GROUP[name]
        if g not in xs:
            if name == "down_proj":  # SiLU(g) * u, g, u ~ N(0, 1) (model.cpp:122-126)
                gz, uz = rng.standard_normal(n), rng.standard_normal(n)
                x = gz / (1 + np.exp(-gz)) * uz
            else:  # heavy-tailed (Laplace x LogNormal)
                x = rng.laplace(size=n) * rng.lognormal(size=n)
            xs[g] = np.ascontiguousarray(x, dtype=np.float64)
    # decoder layers stay resident across passes when host memory allows
    # (~2 GB of fp64 per layer); otherwise each layer is rebuilt per pass
    # (untimed) with only one layer resident at a time
    per_layer = sum(8 * (m * n + r * (m + n)) for (_, m, n, _, r) in plans[:7])
    avail = host_info().get("MemAvailable", 0)
    resident = avail > 1.5 * per_layer * n_layers + (8 << 30)
    cache = {}

    def build(L):
        objs = []
        for (name, m, n, s, r) in plans[7 * L: 7 * L + 7]:
            w, a, b = src[(m, n)]
            a, b = np.ascontiguousarray(a[:, :r]), np.ascontiguousarray(b[:r])
            objs.append(R.layer(w, a, b, s) if use_ref else (w, a, b, s))
        return objs

    ys = {i: np.empty(p[1]) for i, p in enumerate(REF_SHAPES)}
    times = []
    t_end = time.perf_counter() + (seconds or 0.0)
    npass = 0
    while True:
        done = npass - max(warmup, 0)
        if passes is not None and done >= passes:
            break
        if passes is None and done >= 1 and time.perf_counter() >= t_end:
            break
        tok = 0.0
        for L in range(n_layers):
            objs = cache.get(L) or build(L)
            if resident:
                cache[L] = objs
            lin = plans[7 * L: 7 * L + 7]
            for g in range(4):
                idx = [i for i, p in enumerate(lin) if REF_GROUP[p[0].rsplit(".", 1)[1]] == g]
                t0 = time.perf_counter()
                if use_ref:
                    R.forward_many([objs[i] for i in idx], [xs[g]] * len(idx), [ys[i] for i in idx],
                                   min(threads, len(idx)))
                else:
                    R.forward_many([objs[i] for i in idx], [xs[g]] * len(idx), min(threads, len(idx)))
                tok += time.perf_counter() - t0
            del objs
        if npass >= max(warmup, 0):
            times.append(tok)
        npass += 1
    cache.clear()
    tok_s = float(np.median(times))
    hi = host_info()
    return {
        "value": tok_s * 1e6, "unit": "us/token", "cores": min(threads, 3),
        "kind": "reference" if use_ref else "port",
        "sample": (f"{'reference rsparse::forward (oracle/_ref, fp64, -O3)' if use_ref else 'C port (oracle)'}: "
                   f"one decode token through {n_layers} decoder layer(s) x 7 linears of the config-2 plans "
                   f"per pass, "
                   + (f"linears of one input group concurrent on up to {min(threads, 3)} threads, groups sequential"
                      if threads > 1 else "single-threaded, every linear in decode order")
                   + f"; median of {len(times)} passes; "
                   f"host {hi.get('cpu_model', '?')}, nproc {hi.get('nproc')}"),
        "passes": len(times), "pass_times_s": times, "host": hi, "layers_timed": n_layers,
        "resident": resident,
    }


REF_S_PER_LAYER = 0.06  # measured: ~1.8 s per 32-layer token on the GPU box's host (profiles/r02b_bench_reference.json)
REF_BUDGET_S = 240.0


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle.oracle import c_oracle, ref_available, ref_oracle
    R = ref_oracle() if ref_available() else c_oracle()
    plans = ref_config2_plans(R, n_layers=args.layers)
    threads = os.cpu_count() or 1
    t_run = time.perf_counter()
    ref_layers = args.ref_layers
    if ref_layers is None and args.steps * REF_S_PER_LAYER * args.layers > REF_BUDGET_S:
        # keep the run within a few minutes: each step a bounded sample (the
        # first decoder layers of the stack), scaled to the whole stack below
        ref_layers = max(1, int(REF_BUDGET_S / (args.steps * REF_S_PER_LAYER)))
    res = cpu_reference_leg(plans, threads, warmup=min(args.warmup, 1), passes=args.steps, layers=ref_layers)
    scale = args.layers / ref_layers if ref_layers else 1.0
    if scale != 1.0:
        res["value"] *= scale
        res["sample"] += f"; x{scale:g} from {ref_layers} to {args.layers} layers (bounded sample for --steps {args.steps})"
    line = {
        "metric": METRIC, "impl": "reference", "value": res["value"], "unit": "us/token",
        "n_gpus": world, "steps": args.steps, "warmup": min(args.warmup, 1),
        "ms_per_step": res["value"] / 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config2: 32-layer Llama-2-7B-shaped R-Sparse linear stack, batch 1, "
                               "50% model-level sparsity (rho~U(0.3,0.7), C=0.5)",
                   "global_batch": 1, "layers": args.layers, "linears": 7 * args.layers,
                   "layers_timed_per_step": ref_layers or args.layers},
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": res["value"], "unit": "us/token", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host": res["host"], "timed_seconds": sum(res["pass_times_s"]),
        "wall_seconds": time.perf_counter() - t_run,
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
    layers, xs_host, gid, wait = build_stack(rsp, wl, plans, rank, world, dev, torch, args.deterministic)

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
    elif args.exchange == "kernel":
        # row-sharded linears in ONE persistent launch per rank and token; each
        # CTA stores its rows into every rank's full y (CUDA IPC peer memory)
        # and publishes them on every rank's exchange words -- no collective
        from paper_2504_19449_b200.sharding import PeerStack, _CudaArray
        st = PeerStack(layers, xs, wait_prev=wait, device=local)
        launch = lambda: st.launch(stream)  # noqa: E731
        y_dev = torch.as_tensor(_CudaArray(st.base, st.xoff // 4, "<f4"), device=dev)  # every full y
        y_host = torch.empty_like(y_dev, device="cpu").pin_memory()
        ys = [st.full_y(i) for i in range(len(layers))]
    else:
        # row-sharded linears, each followed by one in-place NCCL all-gather
        # of y (paper_2504_19449_b200/sharding.py), captured as one graph
        from paper_2504_19449_b200.sharding import ShardedGroupStack, ShardedStack, even_shards
        if all(even_shards(l.m_out, world) for l in layers) and not os.environ.get("RSP_PER_LINEAR_SHARDS"):
            st = ShardedGroupStack(layers, xs, ys, gid, stream=stream,  # one stack launch per input group
                                   force_gather=args.force_sharded)
        else:
            st = ShardedStack(layers, xs, ys, stream=stream, force_gather=args.force_sharded)
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

    bytes_step = algorithmic_bytes(layers)  # this rank's algorithmic bytes (SURVEY model)
    kbytes_step = kernel_bytes(layers)
    hbm_peak, peak_kind = measured_peaks()
    achieved = bytes_step / (ms_step * 1e-3) / 1e9

    # ---- end to end: H2D of the token's activations, the stack, D2H of all outputs ----
    h2d = x_host.numel() * 2
    d2h = y_dev.numel() * 4

    if not sharded:
        # through the ABI's host-buffer entry (rsp_stack_launch_host): H2D of
        # the token's activations, the stack, D2H of every output, synchronised
        assert st.io_spans() == (x_host.numel() * 2, y_host.numel() * 4)

        def e2e_step():
            st.launch_host(x_host, y_host, stream)
    else:
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
    if args.check and rank == 0:  # the stack's own outputs, before the dense baselines reuse ys
        extras["check"] = check_outputs(layers, xs, ys, plans)
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
                   "parallelism": f"row-shard{world}" + (("+kernel-exchange" if args.exchange == "kernel"
                                                             else "+allgather") if sharded else ""),
                   "combine": "deterministic (fixed-order partials)" if args.deterministic else "float reductions at L2",
                   "sharded_graph": (getattr(st, "graph", None) is not None) if sharded else None,
                   "l2": "no flush: 16 GB resident operands >> 126 MB L2",
                   "activations": "pre-filled synthetic x per input group; stack dependencies (wait_prev) keep "
                                  "the decoder-layer order but y is not fed forward (model.DecodeBlock does that)",
                   "step_ms_p10_p50_p90": [float(np.percentile(per, q)) for q in (10, 50, 90)]},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": None if sharded else load_traffic(),
                     "peak_kind": peak_kind, "algorithmic_bytes_per_step": bytes_step,
                     "kernel_bytes_per_step": kbytes_step,
                     "kernel": ("stack_kernel<bf16,bf16> (1 persistent launch/step, y stored into every rank)"
                                if sharded and args.exchange == "kernel" else
                                "stack_kernel<bf16,bf16> (1 launch per input group, + NCCL all-gather of y)" if sharded
                                else "stack_kernel<bf16,bf16> (1 persistent launch/step, 224 linears)")},
        "e2e": {"value": e2e_ms * 1e3, "unit": "us/token", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "path": "rsp_stack_launch_host (C ABI, pinned host buffers, synchronised per token)" if not sharded
                else "torch pinned copies around the sharded graph"},
        "gpu_launches": args.steps * (max(gid) + 1 if sharded and args.exchange == "nccl" else 1),
        "clocks": clocks.summary(),
    }
    out.update(extras)
    if "dense_cublas_us_per_token" in out:
        out["speedup_vs_dense_cublas"] = out["dense_cublas_us_per_token"] / us_token
        out["speedup_vs_dense_inhouse"] = out["dense_inhouse_us_per_token"] / us_token
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        # single-threaded, as the reference runs (no internal threading,
        # layer.cpp:95-123); the --impl reference arm times the
        # whole stack with its input groups on concurrent threads
        cpu = cpu_reference_leg(plans, 1, seconds=args.cpu_seconds, layers=args.cpu_layers)
        # per-token time of the sampled layers, scaled to the stack (a
        # reported baseline only)
        scale = len(plans) / (7 * cpu["layers_timed"])
        out["cpu_baseline"] = {"value": cpu["value"] * scale, "unit": "us/token", "cores": cpu["cores"],
                               "kind": cpu["kind"],
                               "sample": cpu["sample"] + f"; x{scale:g} from {cpu['layers_timed']} to "
                                                         f"{len(plans) // 7} layers"}

    if rank == 0:
        print(json.dumps(out), flush=True)
    if sharded:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


def check_outputs(layers, xs, ys, plans, every=16):
    """Oracle check of the stack's last outputs (run after the timed loop, not
    timed): for every `every`-th linear and every linear with r > 1024 the
    selection must equal top_k_by_magnitude and y must match the reference
    forward on the device-held values within 1e-5 (max-norm relative)."""
    from oracle.oracle import c_oracle
    C = c_oracle()
    idx = sorted(set(range(0, len(layers), every)) | {i for i, p in enumerate(plans) if p[4] > 1024})
    worst, bad = 0.0, []
    for i in idx:
        l = layers[i]
        W, A, B = l.export()
        x = xs[i].float().cpu().numpy().astype(np.float64)
        yo, kept = C.forward(np.ascontiguousarray(W.T), A, B, plans[i][3], x, return_kept=True)
        yi = ys[i][l.row_begin:l.row_end] if ys[i].numel() == l.m_out else ys[i]  # a rank's own rows
        y = yi.cpu().numpy().astype(np.float64)
        e = float(np.max(np.abs(y - yo)) / max(np.max(np.abs(yo)), 1e-300))
        worst = max(worst, e)
        if e > 1e-5 or not np.array_equal(l.selected(xs[i]), kept):
            bad.append(plans[i][0])
    return {"linears_checked": len(idx), "max_rel_err": worst, "failed": bad, "ok": not bad}


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
