"""Multi-GPU host logic on the CPU: world_size-2 gloo process groups.

The row-sharded path is: every rank selects on the
replicated x, computes the output rows it owns, and one all-gather per
linear reassembles y.  Here each rank's row block is computed by the oracle
(the checker) on exactly the rows rsp_shard_rows assigns, and the product's
gather_rows assembles them; the result must equal the UNSHARDED oracle
forward bit for bit (row i of y depends only on row i of W and A_r and on
the replicated selection).  The device kernels themselves are covered by
tests/test_gpu_parity.py::test_shards_concatenate_to_full.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _operands(m, n, r, seed):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((m, n))
    a = rng.standard_normal((m, r))
    b = rng.standard_normal((r, n))
    x = rng.laplace(size=n) * rng.lognormal(size=n)
    x[rng.choice(n, 3, replace=False)] *= 20
    return w, a, b, x


def _worker(rank, world, port, cases, errq):
    try:
        sys.path.insert(0, ROOT)
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle.oracle import c_oracle
        from paper_2504_19449_b200.sharding import gather_rows, shard_spans
        C = c_oracle()
        for (m, n, r, s, seed, batch) in cases:
            w, a, b, x = _operands(m, n, r, seed)
            b0, e0 = shard_spans(m, world)[rank]
            xs = [x] if batch == 0 else [x * (t + 1) - t for t in range(batch)]
            locs, fulls = [], []
            for xv in xs:
                y_loc, kept = C.forward(np.ascontiguousarray(w[b0:e0].T), a[b0:e0], b, s, xv,
                                        return_kept=True)
                y_full, kept_full = C.forward(np.ascontiguousarray(w.T), a, b, s, xv, return_kept=True)
                assert np.array_equal(kept, kept_full)  # selection is replicated, not sharded
                locs.append(y_loc)
                fulls.append(y_full)
            if batch == 0:
                got = gather_rows(torch.from_numpy(locs[0]), m)
                want = fulls[0]
            else:
                got = gather_rows(torch.from_numpy(np.stack(locs)), m)
                want = np.stack(fulls)
            assert got.shape == want.shape, (got.shape, want.shape)
            assert np.array_equal(got.numpy(), want), (m, n, r, s, batch)
            # every rank holds the identical full output
            chk = torch.tensor([float(np.sum(got.numpy()))], dtype=torch.float64)
            allv = [torch.zeros_like(chk) for _ in range(world)]
            dist.all_gather(allv, chk)
            assert all(torch.equal(allv[0], v) for v in allv)
        dist.destroy_process_group()
    except BaseException as e:  # surface the failure in the parent
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


def _run(world, cases):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]


def test_row_shards_gather_to_unsharded_forward_world2():
    cases = [
        (64, 48, 8, 0.5, 1, 0),      # even shards: all_gather_into_tensor
        (37, 29, 5, 0.33, 2, 0),     # uneven shards: padded gather
        (40, 50, 0, 0.25, 3, 0),     # no low-rank term
        (24, 30, 6, 0.5, 4, 3),      # (batch, rows) block
        (33, 64, 4, 0.77, 5, 2),     # uneven + batch
    ]
    _run(2, cases)


def test_row_shards_world3_uneven():
    _run(3, [(11, 16, 3, 0.5, 6, 0), (100, 40, 7, 0.4, 7, 2)])


def test_shard_spans_match_abi_partition():
    from paper_2504_19449_b200.sharding import shard_spans
    for m in (4096, 11008, 14336, 1024, 37):
        for g in (1, 2, 4, 8):
            spans = shard_spans(m, g)
            assert spans[0][0] == 0 and spans[-1][1] == m
            if m % g == 0:
                assert all(e - b == m // g for (b, e) in spans)


def test_gather_rows_single_process_is_identity():
    from paper_2504_19449_b200.sharding import gather_rows
    y = torch.arange(7, dtype=torch.float32)
    assert torch.equal(gather_rows(y, 7), y)


# ---------------------------------------------------------------- cross-process in-kernel exchange: host logic
class _FakeIpc:
    """Stand-in for the CUDA IPC calls: every process has its own fake
    address space, a peer's area maps at a different address than its own."""

    def __init__(self, rank):
        self.rank, self.opened, self.freed = rank, [], []

    def alloc(self, device, nbytes):
        self.nbytes = nbytes
        return 0x7F00_0000_0000 + self.rank * 0x1_0000_0000

    def export(self, ptr):
        import struct
        return struct.pack("<QQ", ptr, self.nbytes).ljust(64, b"\0")

    def open(self, device, handle):
        import struct
        ptr, _ = struct.unpack("<QQ", handle[:16])
        mapped = ptr + ((self.rank + 1) << 40)  # the peer's area as this process sees it
        self.opened.append(mapped)
        return mapped

    def close(self, ptr):
        pass

    def free(self, ptr):
        self.freed.append(ptr)


class _ShardStub:
    def __init__(self, m, rank, world):
        from paper_2504_19449_b200.sharding import shard_rows
        self.m_out = m
        self.row_begin, self.row_end = shard_rows(m, rank, world)


def _peer_worker(rank, world, port, errq):
    try:
        sys.path.insert(0, ROOT)
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2504_19449_b200.sharding import PeerStack, exchange_layout, plans_agree
        ms = [4096, 1024, 11008, 4096, 37]
        layers = [_ShardStub(m, rank, world) for m in ms]
        ipc = _FakeIpc(rank)
        ps = PeerStack(layers, [0, 0, 1, 2, 3], group=None, ipc=ipc, create=False)
        offs, xoff, nbytes = exchange_layout(ms)
        assert ps.y_offs == offs and ps.xoff == xoff and ipc.nbytes == nbytes
        assert all(o % 16 == 0 for o in offs) and xoff % 256 == 0 and xoff >= offs[-1] + 4 * ms[-1]
        assert nbytes >= xoff + 8 * (len(ms) + 1)  # one word per linear slot + the start fence
        own = 0x7F00_0000_0000 + rank * 0x1_0000_0000
        for p in range(world):  # own area unmapped, peers at their mapped addresses
            want = own if p == rank else 0x7F00_0000_0000 + p * 0x1_0000_0000 + ((rank + 1) << 40)
            assert ps.bases[p] == want, (p, hex(ps.bases[p]), hex(want))
        assert ps.xctr == [b + xoff for b in ps.bases]
        for i, l in enumerate(layers):
            assert ps.y_devs[i] == own + offs[i] + 4 * l.row_begin
            assert ps.y_peers[i] == [b + offs[i] + 4 * l.row_begin for b in ps.bases]
        # x given as "full output of linear j" resolves into the own area
        assert ps.x_devs == [own + offs[j] for j in (0, 0, 1, 2, 3)]
        # across ranks: every destination's rows are partitioned exactly (no gap, no overlap)
        mine = [(ps.y_peers[i][p] - ps.bases[p] - offs[i]) // 4 for i in range(len(ms)) for p in range(world)]
        allr = [None] * world
        dist.all_gather_object(allr, (rank, [(l.row_begin, l.row_end) for l in layers], mine))
        for i, m in enumerate(ms):
            spans = sorted(r[1][i] for r in allr)
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            for rk, sp, mm in allr:  # each rank writes its first row at the same offset in every copy
                assert mm[i * world:(i + 1) * world] == [sp[i][0]] * world
        # plan agreement: equal grids pass, a rank with a different plan fails everywhere
        plans_agree([148, 66, 66])
        try:
            plans_agree([148, 66, 66 + rank])
            raised = False
        except RuntimeError:
            raised = True
        assert raised
        ps.close()
        assert ipc.freed == [own]
        dist.destroy_process_group()
    except BaseException as e:
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


@pytest.mark.parametrize("world", [2, 3])
def test_peer_stack_exchange_tables_world(world):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
