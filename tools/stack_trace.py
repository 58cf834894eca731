"""Per-linear phase timeline inside ONE persistent stack launch
(rsp_debug_stack_trace) for the first decoder layers of the config-2 stack.

    python tools/stack_trace.py [--layers 2] [--mhz 1965]
"""
import argparse
import ctypes as ct
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2504_19449_b200 as rsp  # noqa: E402
from paper_2504_19449_b200 import _lib as L  # noqa: E402
from paper_2504_19449_b200 import workloads as wl  # noqa: E402

PH = {1: "setup", 2: "x+hist", 3: "cut", 4: "lists", 10: "opwait", 11: "s1rows", 12: "treds", 5: "arrive", 6: "Wrows",
      7: "bwait", 8: "Arows", 9: "yred"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--mhz", type=float, default=1965.0)
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--ungrouped", action="store_true")
    ap.add_argument("--det", action="store_true", help="deterministic (atomic-free) combines")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    plans = wl.config2_plans(n_layers=args.layers)
    gid, wait = wl.input_groups(plans)
    rng = np.random.default_rng(0)
    layers, xs, xg = [], [], {}
    for i, (name, m, n, s, r) in enumerate(plans):
        w = torch.randn(m, n, device=dev, dtype=torch.bfloat16) * 0.02
        a = torch.randn(m, r, device=dev, dtype=torch.bfloat16) * 0.05
        b = torch.randn(r, n, device=dev, dtype=torch.bfloat16) * 0.05
        layers.append(rsp.DecomposedLayer(w, a, b, rsp.SparsityPlan(s, r), deterministic=args.det))
        if gid[i] not in xg:
            xg[gid[i]] = torch.from_numpy(wl.heavy_tailed_x(n, rng)).to(dev).to(torch.bfloat16)
        xs.append(xg[gid[i]])
    ys = [torch.empty(l.m_out, device=dev) for l in layers]
    st = rsp.Stack(layers, xs, ys, dense=args.dense, wait_prev=None if args.ungrouped else wait)
    for _ in range(5):
        st.launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        st.launch()
    e1.record()
    e1.synchronize()
    print(f"stack of {len(layers)} linears: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per launch "
          f"({e0.elapsed_time(e1) / 20 * 1e3 / len(layers):.2f} us per linear)")
    grid = ct.c_uint32()
    tr = torch.zeros(len(layers) * 148 * 16, dtype=torch.int64, device=dev)
    for _ in range(3):
        tr.zero_()
        L.check(L.lib().rsp_debug_stack_trace(st._h, tr.data_ptr(), ct.byref(grid), None))
    torch.cuda.synchronize()
    G = grid.value
    t = tr[: len(layers) * G * 16].view(len(layers), G, 16).cpu().numpy()
    t0 = t[0, :, 0].min()
    prev_end = t0
    print("linear            grid  start  waitd   end   wall | phase medians (us, cumulative from run start)")
    for i, (name, m, n, s, r) in enumerate(plans):
        part = t[i, :, 1] > 0  # CTAs that worked on this linear
        g = int(part.sum())
        start = (t[i, :, 0].min() - t0) / 1e3
        waitd = (np.median(t[i, :, 13]) - t0) / 1e3
        end = (t[i, :, 14].max() - t0) / 1e3
        wall = (t[i, :, 14].max() - prev_end) / 1e3
        prev_end = t[i, :, 14].max()
        ph = []
        for ev, lab in PH.items():
            col = t[i, part, ev]
            col = col[col > 0]
            if col.size:
                ph.append(f"{lab}={np.median(col) / args.mhz:.2f}")
        print(f"{name.split('.', 1)[1]:17s} {g:4d} {start:6.2f} {waitd:6.2f} {end:6.2f} {wall:6.2f} | " + " ".join(ph))
    # finish spread: absolute time each CTA issued its last y reduction
    # (dependency-wait stamp + run-relative yred clock), and when the next
    # group's CTAs saw their dependency satisfied
    print("linear            finish median/p90/max (us from launch start) | next waitd min/median")
    for i, (name, m, n, s, r) in enumerate(plans):
        part = t[i, :, 1] > 0
        fin = (t[i, part, 13] - t0) / 1e3 + t[i, part, 9] / args.mhz
        nxt = ""
        for j in range(i + 1, len(plans)):
            pj = t[j, :, 1] > 0
            if pj.any():
                w = (t[j, pj, 13] - t0) / 1e3
                nxt = f"{name.split('.', 1)[1]} -> {plans[j][0].split('.', 1)[1]}: {w.min():6.2f} / {np.median(w):6.2f}"
                break
        print(f"{name.split('.', 1)[1]:17s} {np.median(fin):6.2f} / {np.percentile(fin, 90):6.2f} / {fin.max():6.2f} | {nxt}")
    for i in range(min(7, len(plans))):
        print(f"stragglers of linear {i} ({plans[i][0]}):")
        stragglers(t, i, args.mhz)


def stragglers(t, i, mhz, top=6):
    """Phase stamps (us from the CTA's run start) of the CTAs finishing linear i last."""
    part = t[i, :, 1] > 0
    idx = np.where(part)[0]
    end = t[i, idx, 14]
    order = idx[np.argsort(end)[::-1][:top]]
    med = {ev: np.median(t[i, idx, ev]) / mhz for ev in PH}
    nw = t[i, idx, 15] & 0xffffffff
    nu = t[i, idx, 15] >> 32
    print(f"  median: nW={np.median(nw):.0f} (min {nw.min()}, max {nw.max()}) nU={np.median(nu):.0f} (max {nu.max()}) | "
          + " ".join(f"{PH[ev]}={med[ev]:.2f}" for ev in PH))
    fin = t[i, idx, 9]
    print(f"  corr(finish, nW) = {np.corrcoef(fin, nw)[0, 1]:.2f}  corr(finish, nU) = {np.corrcoef(fin, nu)[0, 1]:.2f}")
    t0 = t[i, idx, 0].min()
    for c in order:
        print(f"  cta {c:3d} nW={t[i, c, 15] & 0xffffffff} nU={t[i, c, 15] >> 32} end={(t[i, c, 14] - t0) / 1e3:6.2f} start={(t[i, c, 0] - t0) / 1e3:5.2f} waitd={(t[i, c, 13] - t0) / 1e3:5.2f} | "
              + " ".join(f"{PH[ev]}={t[i, c, ev] / mhz:.2f}" for ev in PH))


if __name__ == "__main__":
    main()
