"""Seeded random sweeps of the sm_100a path against the oracle.

The fixed-shape parity tests (test_gpu_parity.py, test_gpu_config2.py) pin
the reference's configurations; these sweeps draw shapes, ranks, keep
fractions, dtypes and activation distributions at random so that the
planner's partitions (k-splits, CTA groups, the C1 stage-1 warp maps, the
list capacities) are hit in combinations no hand-written case names.  Every
case is checked the same way as the parity suite: the selected set
bit-exact and y within TOL_EXACT_INPUTS of the oracle run on the values the
device holds (rsparse::forward, layer.cpp:95-123).
"""
import numpy as np
import pytest
import torch

import paper_2504_19449_b200 as rsp
from paper_2504_19449_b200 import workloads as wl
from paper_2504_19449_b200._lib import RSP_E_UNSUPPORTED

from test_gpu_parity import TOL_EXACT_INPUTS, maxrel, oracle_on_device_values

pytestmark = pytest.mark.gpu


def random_x(rng, n):
    """One of several activation distributions, ties and zeros included."""
    kind = rng.integers(0, 5)
    if kind == 0:
        x = wl.heavy_tailed_x(n, rng, outliers=min(8, n))
    elif kind == 1:
        x = rng.standard_normal(n)
    elif kind == 2:  # coarse levels: many exact ties in |x|, resolved by lower index
        x = np.round(rng.standard_normal(n) * 2.0) / 2.0
    elif kind == 3:  # mostly zeros
        x = rng.standard_normal(n) * (rng.random(n) < 0.2)
    else:
        x = wl.silu_gate_x(n, rng)
    return np.asarray(x, np.float32)


def random_linear(rng, cuda, wdt, m=None, n=None, det=None):
    m = int(m or rng.integers(1, 9000))
    n = int(n or rng.integers(1, 9000))
    # B_r^T rows of at most 4 KB (rsp_linear_create's documented limit)
    r_max = 2048 if wdt == "bf16" else 1024
    r = int(min(m, n, r_max, rng.choice([0, 1, 7, 64, 255, 256, 513, 1024, 1025, 1100, 2048])))
    s = float(rng.choice([0.0, 1.0, rng.random(), rng.random(), rng.random()]))
    w = torch.randn(m, n, device=cuda) * 0.02
    a = torch.randn(m, r, device=cuda) * 0.1
    b = torch.randn(r, n, device=cuda) * 0.1
    if det is None:
        det = bool(rng.random() < 0.2)
    return rsp.DecomposedLayer(w, a, b, rsp.SparsityPlan(s, r), weight_dtype=wdt, deterministic=det)


@pytest.mark.parametrize("seed", range(6))
def test_forward_random_configs(coracle, cuda, seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(8):
        wdt = str(rng.choice(["f32", "bf16"]))
        xdt = str(rng.choice(["f32", "bf16"]))
        layer = random_linear(rng, cuda, wdt)
        xt = torch.from_numpy(random_x(rng, layer.m_in)).to(cuda)
        xt = xt.to(torch.bfloat16) if xdt == "bf16" else xt
        y = layer.forward(xt).cpu().numpy()
        yo, kept, _ = oracle_on_device_values(coracle, layer, xt)
        tag = (layer.m_out, layer.m_in, layer.plan.rank, layer.plan.keep_fraction, wdt, xdt)
        assert np.array_equal(layer.selected(xt), kept), tag
        assert maxrel(y, yo) <= TOL_EXACT_INPUTS, (tag, maxrel(y, yo))


@pytest.mark.parametrize("seed", range(4))
def test_stack_random_configs(coracle, cuda, seed):
    """A random persistent stack: random shapes, ranks and keep fractions,
    random sharing of inputs (wait_prev False) and dependencies."""
    rng = np.random.default_rng(2000 + seed)
    wdt, xdt = [("bf16", "bf16"), ("f32", "f32"), ("bf16", "f32"), ("f32", "bf16")][seed]
    count = int(rng.integers(5, 13))
    det = seed == 3  # a stack runs in one combine mode (rsp_stack_create rejects a mix)
    layers, xs, wait = [], [], []
    for i in range(count):
        share = i > 0 and rng.random() < 0.35
        n = layers[-1].m_in if share else None
        layers.append(random_linear(rng, cuda, wdt, n=n, det=det))
        if share:
            xs.append(xs[-1])
        else:
            xt = torch.from_numpy(random_x(rng, layers[-1].m_in)).to(cuda)
            xs.append(xt.to(torch.bfloat16) if xdt == "bf16" else xt)
        wait.append(not share)
    ys = [torch.full((l.m_out,), float("nan"), device=cuda) for l in layers]
    st = rsp.Stack(layers, xs, ys, wait_prev=wait)
    for _ in range(2):
        st.launch()
    torch.cuda.synchronize()
    for i, (l, x, y) in enumerate(zip(layers, xs, ys)):
        yo, _, _ = oracle_on_device_values(coracle, l, x)
        got = y.cpu().numpy()
        assert np.isfinite(got).all(), i
        assert maxrel(got, yo) <= TOL_EXACT_INPUTS, (i, l.m_out, l.m_in, l.plan.rank, maxrel(got, yo))


def test_rank_limit_is_unsupported_not_wrong(cuda):
    """Ranks whose B_r^T row exceeds 4 KB are refused at create time with
    RSP_E_UNSUPPORTED (documented in rsp_linear_create), never run."""
    m, n = 2100, 2100
    for wdt, r in (("f32", 1025), ("bf16", 2049)):
        w = torch.randn(m, n, device=cuda)
        with pytest.raises(rsp.RspError) as e:
            rsp.DecomposedLayer(w, torch.randn(m, r, device=cuda), torch.randn(r, n, device=cuda),
                                rsp.SparsityPlan(0.5, r), weight_dtype=wdt)
        assert e.value.status == RSP_E_UNSUPPORTED


@pytest.mark.parametrize("max_ctas", [0, 8])
def test_stack_group_minimum_partitions(coracle, cuda, max_ctas):
    """Input-sharing group members whose byte share is tiny (s = 0, r = 0
    moves no weight bytes) still get the CTAs their column tiling needs; a
    group whose minimums exceed the launch budget (max_ctas = 8 against
    3 x 4 CTAs) is split and run in order."""
    rng = np.random.default_rng(77)
    n = 3000
    shapes = [(4096, 0.4, 256), (4096, 0.0, 0), (3813, 0.7, 100)]
    layers = [rsp.DecomposedLayer(torch.randn(m, n, device=cuda) * 0.02, torch.randn(m, r, device=cuda) * 0.1,
                                  torch.randn(r, n, device=cuda) * 0.1, rsp.SparsityPlan(s, r), weight_dtype="f32")
              for (m, s, r) in shapes]
    x = torch.from_numpy(wl.heavy_tailed_x(n, rng)).to(cuda)
    ys = [torch.full((l.m_out,), float("nan"), device=cuda) for l in layers]
    st = rsp.Stack(layers, [x] * 3, ys, wait_prev=[True, False, False], max_ctas=max_ctas)
    st.launch()
    torch.cuda.synchronize()
    for l, y in zip(layers, ys):
        yo, _, _ = oracle_on_device_values(coracle, l, x)
        assert maxrel(y.cpu().numpy(), yo) <= TOL_EXACT_INPUTS


def test_forward_host_concurrent_threads(coracle, cuda):
    """forward is re-entrant in the reference; the host-buffer
    entry point on ONE handle from several threads (ctypes drops the GIL)
    must give every caller its own token's result."""
    import threading
    rng = np.random.default_rng(5)
    m, n, r = 2048, 3072, 128
    layer = rsp.DecomposedLayer(torch.randn(m, n, device=cuda) * 0.02, torch.randn(m, r, device=cuda) * 0.1,
                                torch.randn(r, n, device=cuda) * 0.1, rsp.SparsityPlan(0.4, r),
                                deterministic=True)  # bit-reproducible, so any mix-up shows
    xs = [wl.heavy_tailed_x(n, rng) for _ in range(8)]
    want = [layer.forward_host(x) for x in xs]
    got = [None] * len(xs)

    def work(t):
        for _ in range(20):
            i = (t * 3 + _) % len(xs)
            y = layer.forward_host(xs[i])
            if not np.array_equal(y, want[i]):
                got[t] = i
                return
        got[t] = -1

    threads = [threading.Thread(target=work, args=(t,)) for t in range(len(xs))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert got == [-1] * len(xs)
    yo, _, _ = oracle_on_device_values(coracle, layer, torch.from_numpy(xs[0]).to(cuda))
    assert maxrel(want[0], yo) <= TOL_EXACT_INPUTS


@pytest.mark.parametrize("xdt", ["f32", "bf16"])
def test_misaligned_inputs_and_outputs(coracle, cuda, xdt):
    """x and y that are not 16-byte aligned (views one element into a buffer)
    take the scalar load / store paths of the selector and the combine."""
    rng = np.random.default_rng(31)
    m, n, r = 1000, 2056, 96
    layers = [rsp.DecomposedLayer(torch.randn(m, n, device=cuda) * 0.02, torch.randn(m, r, device=cuda) * 0.1,
                                  torch.randn(r, n, device=cuda) * 0.1, rsp.SparsityPlan(s, r)) for s in (0.3, 0.6)]
    buf = torch.from_numpy(random_x(rng, n + 1)).to(cuda)
    buf = buf.to(torch.bfloat16) if xdt == "bf16" else buf
    x = buf[1:]  # 2 or 4 bytes past a 16-byte boundary
    ybuf = torch.full((2 * m + 2,), float("nan"), device=cuda)
    ys = [ybuf[1:1 + m], ybuf[1 + m:1 + 2 * m]]
    for l in layers:
        yo, kept, _ = oracle_on_device_values(coracle, l, x)
        assert np.array_equal(l.selected(x), kept)
        assert maxrel(l.forward(x).cpu().numpy(), yo) <= TOL_EXACT_INPUTS
    st = rsp.Stack(layers, [x, x], ys, wait_prev=[True, False])
    st.launch()
    torch.cuda.synchronize()
    for l, y in zip(layers, ys):
        yo, _, _ = oracle_on_device_values(coracle, l, x)
        assert maxrel(y.cpu().numpy(), yo) <= TOL_EXACT_INPUTS


def test_widest_inputs(coracle, cuda):
    """m_in up to 32768: with bf16 activations x stays on chip as bf16;
    fp32 activations that no longer fit are refused (RSP_E_UNSUPPORTED),
    not computed wrongly.  28000 channels still take fp32."""
    rng = np.random.default_rng(3)
    for n, f32_ok in ((28000, True), (32768, False)):
        m, r = 256, 64
        l = rsp.DecomposedLayer(torch.randn(m, n, device=cuda) * 0.02, torch.randn(m, r, device=cuda) * 0.1,
                                torch.randn(r, n, device=cuda) * 0.1, rsp.SparsityPlan(0.3, r))
        x32 = torch.from_numpy(random_x(rng, n)).to(cuda)
        for x in (x32.to(torch.bfloat16), x32):
            if x.dtype == torch.float32 and not f32_ok:
                with pytest.raises(rsp.RspError) as e:
                    l.forward(x)
                assert e.value.status == RSP_E_UNSUPPORTED
                continue
            yo, kept, _ = oracle_on_device_values(coracle, l, x)
            assert np.array_equal(l.selected(x), kept), (n, x.dtype)
            assert maxrel(l.forward(x).cpu().numpy(), yo) <= TOL_EXACT_INPUTS, (n, x.dtype)
