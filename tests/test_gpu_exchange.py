"""Row-sharded ranks with the y exchange done by the kernel's own stores
(SURVEY 8(e)): each rank's shard CTAs write their output rows into EVERY
rank's copy of the full y (rsp_stack_create_spec, npeer > 1) instead of an
NCCL all-gather after the launch.  One GPU stands in for the ranks the way
the profiling guide prescribes -- one kernel over all ranks' data: every
rank's shards run side by side in ONE persistent launch, each rank with its
own full-length y buffers, and a dependent linear of rank r reads rank r's
copy (the data another rank's CTAs wrote)."""
import numpy as np
import pytest
import torch

import paper_2504_19449_b200 as rsp
from paper_2504_19449_b200 import workloads as wl

pytestmark = pytest.mark.gpu


def maxrel(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return np.max(np.abs(got - want)) / np.max(np.abs(want))


@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_ranks_in_one_launch_exchange_y_in_kernel(cuda, ranks):
    rng = np.random.default_rng(ranks)
    # q: 1536 x 512, k: 512 x 512 (share x), o: 512 x 1536 reads q's full output
    specs = {"q": (1536, 512, 0.3, 48), "k": (512, 512, 0.25, 32), "o": (512, 1536, 0.2, 64)}
    W = {}
    for name, (m, n, s, r) in specs.items():
        W[name] = (torch.randn(m, n, device=cuda) * 0.05, torch.randn(m, r, device=cuda) * 0.1,
                   torch.randn(r, n, device=cuda) * 0.1, rsp.SparsityPlan(s, r))
    full = {k: rsp.DecomposedLayer(*v[:3], v[3], weight_dtype="bf16") for k, v in W.items()}
    shard = {k: [rsp.DecomposedLayer(*v[:3], v[3], weight_dtype="bf16", shard_rank=p, shard_count=ranks)
                 for p in range(ranks)] for k, v in W.items()}
    x = torch.from_numpy(wl.heavy_tailed_x(512, rng)).to(cuda)
    Y = {k: [torch.full((specs[k][0],), float("nan"), device=cuda) for _ in range(ranks)] for k in specs}
    layers, xs, ys, peers, wait = [], [], [], [], []
    for name in ("q", "k", "o"):
        for p in range(ranks):
            l = shard[name][p]
            layers.append(l)
            xs.append(x if name != "o" else Y["q"][p])   # o on rank p reads rank p's copy of q's y
            ys.append(Y[name][p][l.row_begin:l.row_end])
            peers.append([Y[name][d][l.row_begin:] for d in range(ranks)])
            wait.append(name != "k" and p == 0)            # q/k shards share x; o waits for all of them
    st = rsp.Stack(layers, xs, ys, wait_prev=wait, y_peers=peers)
    for _ in range(3):
        st.launch()
    torch.cuda.synchronize()
    want_q, want_k = full["q"].forward(x).cpu().numpy(), full["k"].forward(x).cpu().numpy()
    for p in range(ranks):
        assert torch.isfinite(Y["q"][p]).all() and torch.isfinite(Y["k"][p]).all() and torch.isfinite(Y["o"][p]).all()
        assert maxrel(Y["q"][p].cpu().numpy(), want_q) <= 1e-6
        assert maxrel(Y["k"][p].cpu().numpy(), want_k) <= 1e-6
        # o on the input it actually read (rank p's assembled copy of q's output)
        assert maxrel(Y["o"][p].cpu().numpy(), full["o"].forward(Y["q"][p]).cpu().numpy()) <= 1e-6
    for p in range(1, ranks):  # every rank holds the same assembled outputs (up to float-atomic order)
        assert maxrel(Y["q"][p].cpu().numpy(), Y["q"][0].cpu().numpy()) <= 1e-6


def test_peer_stack_one_rank_counts_and_outputs(cuda):
    """The cross-process path (rsp_stack_spec.xrank) at world size 1 -- the
    only size one GPU can run without ranks whose kernels wait on each other:
    the per-launch start fence, the sys-scope arrivals on the exchange words
    and the cumulative (never reset) dependency targets over many launches.
    o reads q's full output from the exchange area (in-launch dataflow)."""
    from paper_2504_19449_b200.sharding import PeerStack, _CudaArray
    rng = np.random.default_rng(11)
    specs = [(1536, 512, 0.3, 48), (512, 512, 0.25, 32), (512, 1536, 0.2, 64)]
    layers = [rsp.DecomposedLayer(torch.randn(m, n, device=cuda) * 0.05, torch.randn(m, r, device=cuda) * 0.1,
                                  torch.randn(r, n, device=cuda) * 0.1, rsp.SparsityPlan(s, r), weight_dtype="bf16")
              for (m, n, s, r) in specs]
    x = torch.from_numpy(wl.heavy_tailed_x(512, rng)).to(cuda)
    ps = PeerStack(layers, [x, x, 0], wait_prev=[True, False, True])
    launches = 25
    for _ in range(launches):
        ps.launch()
    torch.cuda.synchronize()
    q, k, o = (ps.full_y(i).clone() for i in range(3))
    assert maxrel(q.cpu().numpy(), layers[0].forward(x).cpu().numpy()) <= 1e-6
    assert maxrel(k.cpu().numpy(), layers[1].forward(x).cpu().numpy()) <= 1e-6
    assert maxrel(o.cpu().numpy(), layers[2].forward(q).cpu().numpy()) <= 1e-6
    grids = (rsp._lib.ct.c_uint32 * 3)()
    rsp._lib.check(rsp.lib().rsp_stack_grids(ps._h, grids, 3))
    words = torch.as_tensor(_CudaArray(ps.base + ps.xoff, 4, "<u8"), device=cuda).cpu().tolist()
    # one publication per group and launch (by the CTA completing the group on
    # this rank): {q, k} on q's slot, o on its own; k's word unused; the start fence
    assert words == [launches, 0, launches, launches], (words, list(grids))
    assert all(g > 0 for g in grids)
    ps.close()


def test_peer_stack_spec_errors(cuda):
    from paper_2504_19449_b200 import _lib as L
    l = rsp.DecomposedLayer(torch.randn(256, 256, device=cuda), torch.randn(256, 8, device=cuda),
                            torch.randn(8, 256, device=cuda), rsp.SparsityPlan(0.5, 8))
    x = torch.randn(256, device=cuda)
    y = torch.empty(256, device=cuda)
    ctr = torch.zeros(4, dtype=torch.int64, device=cuda)
    sp = L.StackSpec()
    sp.layers = (L.ct.c_void_p * 1)(l.handle.value)
    sp.count, sp.x_dtype = 1, L.RSP_F32
    sp.x_devs = (L.ct.c_void_p * 1)(x.data_ptr())
    sp.y_devs = (L.ct.c_void_p * 1)(y.data_ptr())
    sp.xrank, sp.xself, sp.npeer = 2, 0, 1  # two ranks but one y destination
    sp.xctr = (L.ct.c_void_p * 2)(ctr.data_ptr(), ctr.data_ptr())
    h = L.ct.c_void_p()
    assert L.lib().rsp_stack_create_spec(L.ct.byref(sp), L.ct.byref(h)) == L.RSP_E_USAGE
    sp.xrank, sp.xself = 1, 1  # xself out of range
    assert L.lib().rsp_stack_create_spec(L.ct.byref(sp), L.ct.byref(h)) == L.RSP_E_USAGE
    d = rsp.DecomposedLayer(torch.randn(256, 256, device=cuda), torch.randn(256, 8, device=cuda),
                            torch.randn(8, 256, device=cuda), rsp.SparsityPlan(0.5, 8), deterministic=True)
    sp.layers = (L.ct.c_void_p * 1)(d.handle.value)
    sp.xself = 0
    assert L.lib().rsp_stack_create_spec(L.ct.byref(sp), L.ct.byref(h)) == L.RSP_E_UNSUPPORTED
