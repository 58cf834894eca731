"""Output-row sharding of the R-Sparse operator across the GPUs of one box.

The reference has no parallelism ("Parallelism strategies");
the north star adds one: every linear's output rows -- the rows of W and of
A_r -- are split over the ranks, B_r (the SVD's V_r side) and x are
replicated, and one all-gather of y per linear reassembles the output
(SURVEY.md §8(e)).  y[i] depends only on row i of W and A_r, and the
selection depends only on x, which every rank holds, so each rank selects
the same channel set and computes exactly the unsharded rows it owns.

Row partition: rank g owns [floor(m*g/G), floor(m*(g+1)/G)) (rsp_shard_rows,
the partition rsp_linear_create applies).  When every shard has the same
length (all BASELINE shapes at G <= 8) each rank's kernel writes straight
into its slot of the full output and the all-gather runs in place, so no
copy surrounds the collective.  Uneven shards go through a padded buffer.

Communication is torch.distributed (NCCL on the GPUs; gloo in the CPU tests
of this host logic).  Compute is librsparse_b200.so.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

from .layer import DecomposedLayer, SparsityPlan, shard_rows

try:
    import torch
    import torch.distributed as dist
except ImportError:  # pragma: no cover
    torch = dist = None


def _group_info(group) -> Tuple[int, int]:
    if dist is None or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def shard_spans(m_out: int, world: int) -> List[Tuple[int, int]]:
    """[(begin, end)] for every rank (host-only; no device needed)."""
    return [shard_rows(m_out, g, world) for g in range(world)]


def even_shards(m_out: int, world: int) -> bool:
    return m_out % world == 0


def gather_rows(y_local, m_out: int, group=None, out=None):
    """All-gather the row shards of one output vector (or a (batch, rows)
    block) into the full (…, m_out) result, in rank order.

    Even shards: one all_gather_into_tensor.  If ``y_local`` already IS the
    caller's slot of ``out`` (the in-place layout ShardedLinear uses), the
    collective runs in place.  Uneven shards: pad to the longest shard,
    gather, then unpad."""
    rank, world = _group_info(group)
    batch_shape = tuple(y_local.shape[:-1])
    if out is None:
        out = y_local.new_empty(batch_shape + (m_out,))
    if world == 1:
        if out.data_ptr() != y_local.data_ptr():
            out.copy_(y_local)
        return out
    spans = shard_spans(m_out, world)
    b, e = spans[rank]
    if y_local.shape[-1] != e - b:
        raise ValueError(f"rank {rank} holds {y_local.shape[-1]} rows, owns {e - b}")
    if not batch_shape and even_shards(m_out, world):
        dist.all_gather_into_tensor(out, y_local.contiguous(), group=group)
        return out
    rows = max(e1 - b1 for (b1, e1) in spans)
    nb = 1
    for d in batch_shape:
        nb *= d
    send = y_local.new_zeros((nb, rows))
    send[:, : e - b] = y_local.reshape(nb, e - b)
    recv = y_local.new_empty((world, nb, rows))
    dist.all_gather_into_tensor(recv.view(-1), send.view(-1), group=group)
    full = out.view(nb, m_out)
    for g, (b1, e1) in enumerate(spans):
        full[:, b1:e1] = recv[g, :, : e1 - b1]
    return out


class ShardedLinear:
    """One R-Sparse linear row-sharded over the ranks of ``group``: this
    rank's DecomposedLayer shard plus the per-linear all-gather of y.

    ``forward(x)`` returns the full fp32 y on every rank (the reference's
    forward(layer, x), layer.cpp:95-123, computed by G GPUs)."""

    def __init__(self, w, a_r=None, b_r=None, plan: Optional[SparsityPlan] = None, *, group=None,
                 device: Optional[int] = None, **kw):
        self.group = group
        self.rank, self.world = _group_info(group)
        if device is None:
            device = torch.cuda.current_device()
        self.layer = DecomposedLayer(w, a_r, b_r, plan, device=device, shard_rank=self.rank,
                                     shard_count=self.world, **kw)
        self.m_in, self.m_out = self.layer.m_in, self.layer.m_out
        self.row_begin, self.row_end = self.layer.row_begin, self.layer.row_end
        self.in_place = even_shards(self.m_out, self.world)

    @classmethod
    def from_layer(cls, layer: DecomposedLayer, group=None) -> "ShardedLinear":
        """Wrap an existing shard (a DecomposedLayer created with
        shard_rank/shard_count of this group) without re-uploading weights."""
        self = cls.__new__(cls)
        self.group = group
        self.rank, self.world = _group_info(group)
        self.layer = layer
        self.m_in, self.m_out = layer.m_in, layer.m_out
        self.row_begin, self.row_end = layer.row_begin, layer.row_end
        self.in_place = even_shards(self.m_out, self.world)
        return self

    def forward(self, x, out=None, workspace=None, stream=None, force_gather: bool = False):
        """force_gather: run the collective on a single rank too (exercises
        the NCCL-in-graph path on one GPU)."""
        if out is None:
            out = torch.empty(self.m_out, dtype=torch.float32, device=x.device)
        if self.in_place and x.dim() == 1:
            mine = out[self.row_begin:self.row_end]
            self.layer.forward(x, out=mine, workspace=workspace, stream=stream)
            if self.world > 1 or (force_gather and dist.is_initialized()):
                dist.all_gather_into_tensor(out, mine, group=self.group)
            return out
        y_local = self.layer.forward(x, workspace=workspace, stream=stream)
        if x.dim() > 1 and out.dim() == 1:
            out = torch.empty((x.shape[0], self.m_out), dtype=torch.float32, device=x.device)
        return gather_rows(y_local, self.m_out, self.group, out=out)

    __call__ = forward


class ShardedStack:
    """A decode-order sequence of sharded linears (forward + all-gather each)
    captured once into a CUDA graph; one replay = one token through the stack.
    ``xs[i]`` / ``ys[i]`` (full-length fp32) are bound at capture time."""

    def __init__(self, linears: Sequence[ShardedLinear], xs, ys, stream=None, group=None,
                 force_gather: bool = False):
        # DecomposedLayer shards (built with shard_rank/shard_count) are wrapped
        self.linears = [l if isinstance(l, ShardedLinear) else ShardedLinear.from_layer(l, group) for l in linears]
        self.xs, self.ys = list(xs), list(ys)
        self.force = force_gather
        self.stream = stream or torch.cuda.Stream()
        # one workspace per linear: the fused kernel's grid barrier words are
        # per-workspace, and consecutive kernels may overlap under PDL
        self.ws = [l.layer.workspace() for l in self.linears]
        with torch.cuda.stream(self.stream):
            self._run()  # warm NCCL communicators outside capture
            torch.cuda.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=self.stream):
                self._run()

    def _run(self):
        for l, x, y, ws in zip(self.linears, self.xs, self.ys, self.ws):
            l.forward(x, out=y, workspace=ws, stream=self.stream, force_gather=self.force)

    def launch(self):
        self.graph.replay()


class ShardedGroupStack:
    """The row-sharded stack with one persistent stack-kernel launch per input
    group (q/k/v, o, gate/up, down) instead of one launch per linear: each
    group's shards run side by side (layer.Stack), then one in-place NCCL
    all-gather per linear assembles the full y on every rank.  All of it is
    captured into one CUDA graph (the stack kernels as plain launches,
    rsp_stack_launch_direct), else replayed eagerly.  Needs even shards (every
    BASELINE shape at N <= 8); `ys[i]` are the full-length outputs."""

    def __init__(self, layers: Sequence[DecomposedLayer], xs, ys, gid: Sequence[int], stream=None, group=None,
                 force_gather: bool = False):
        from .layer import Stack
        self.rank, self.world = _group_info(group)
        self.group = group
        self.stream = stream or torch.cuda.Stream()
        self.layers, self.xs, self.ys = list(layers), list(xs), list(ys)
        for l in self.layers:
            if not even_shards(l.m_out, self.world):
                raise ValueError("ShardedGroupStack needs even row shards")
        self.groups = []
        for g in sorted(set(gid)):
            idx = [i for i in range(len(self.layers)) if gid[i] == g]
            locs = [self.ys[i][self.layers[i].row_begin:self.layers[i].row_end] for i in idx]
            st = Stack([self.layers[i] for i in idx], [self.xs[i] for i in idx], locs,
                       wait_prev=[False] * len(idx))
            self.groups.append((st, idx, locs))
        self.force = force_gather and dist.is_initialized()
        self.graph = None
        with torch.cuda.stream(self.stream):
            self._run()  # warm NCCL communicators outside capture
            torch.cuda.synchronize()
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.stream):
                    self._run()
                self.graph = g
            except RuntimeError:
                torch.cuda.synchronize()
                self.graph = None

    def _run(self):
        for st, idx, locs in self.groups:
            st.launch(self.stream, direct=True)  # capturable into the step's graph with the all-gathers
            if self.world > 1 or self.force:
                for i, loc in zip(idx, locs):
                    dist.all_gather_into_tensor(self.ys[i], loc, group=self.group)

    def launch(self):
        if self.graph is not None:
            self.graph.replay()
        else:
            with torch.cuda.stream(self.stream):
                self._run()

    def close(self):
        for st, _, _ in self.groups:
            st.close()


# ----------------------------------------------------------------------------
# The exchange inside the kernel, across processes (rsp_stack_spec.xrank)
# ----------------------------------------------------------------------------
class IpcOps:
    """The CUDA IPC calls the cross-process exchange needs (rsp_ipc_* in the
    library).  Kept behind one object so that the host logic -- handle
    exchange, address tables, plan agreement -- runs in CPU tests with a
    stand-in (tests/test_sharding.py)."""

    def alloc(self, device: int, nbytes: int) -> int:
        from . import _lib as L
        p = L.ct.c_void_p()
        L.check(L.lib().rsp_ipc_alloc(device, nbytes, L.ct.byref(p)), "rsp_ipc_alloc")
        return int(p.value)

    def export(self, ptr: int) -> bytes:
        from . import _lib as L
        buf = L.ct.create_string_buffer(L.RSP_IPC_HANDLE_BYTES)
        L.check(L.lib().rsp_ipc_export(L.ct.c_void_p(ptr), buf), "rsp_ipc_export")
        return buf.raw

    def open(self, device: int, handle: bytes) -> int:
        from . import _lib as L
        p = L.ct.c_void_p()
        L.check(L.lib().rsp_ipc_open(device, handle, L.ct.byref(p)), "rsp_ipc_open")
        return int(p.value)

    def close(self, ptr: int) -> None:
        from . import _lib as L
        L.lib().rsp_ipc_close(L.ct.c_void_p(ptr))

    def free(self, ptr: int) -> None:
        from . import _lib as L
        L.lib().rsp_ipc_free(L.ct.c_void_p(ptr))


def _align(v: int, a: int = 256) -> int:
    return (v + a - 1) // a * a


def exchange_layout(m_outs: Sequence[int]) -> Tuple[List[int], int, int]:
    """Byte layout of a rank's exchange area, the same on every rank: the
    full fp32 y of every linear (16-B aligned), then the 64-bit exchange
    words (rsp_stack_exchange_words: one arrival word per linear slot, then
    the start fence).  Returns (y offsets, word offset, total bytes)."""
    offs, cur = [], 0
    for m in m_outs:
        offs.append(cur)
        cur = _align(cur + 4 * int(m), 16)
    xoff = _align(cur)
    return offs, xoff, _align(xoff + 8 * (len(m_outs) + 1))


def exchange_tables(bases: Sequence[int], y_offs: Sequence[int], xoff: int,
                    row_begins: Sequence[int]) -> Tuple[List[List[int]], List[int]]:
    """Every linear's y destinations on all ranks (this shard's first row in
    each rank's full y) and every rank's exchange words."""
    y_peers = [[b + off + 4 * rb for b in bases] for off, rb in zip(y_offs, row_begins)]
    return y_peers, [b + xoff for b in bases]


def _all_gather_object(obj, group):
    rank, world = _group_info(group)
    if world == 1:
        return [obj]
    out = [None] * world
    dist.all_gather_object(out, obj, group=group)
    return out


def plans_agree(grids: Sequence[int], group=None) -> None:
    """The dependency targets of a cross-process stack count every rank's
    CTAs as this rank's grid x world: all ranks must have planned the same
    per-linear grids.  Raises on every rank otherwise."""
    allg = _all_gather_object(list(grids), group)
    if any(g != allg[0] for g in allg):
        raise RuntimeError(f"PeerStack: the ranks planned different CTA grids (uneven shards?): {allg}")


class _CudaArray:
    """__cuda_array_interface__ over a raw device range (torch views of the area)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


class PeerStack:
    """One rank's part of a row-sharded stack with one process per GPU and
    the all-gather of y done by the kernel itself (SURVEY 8(e) without a
    collective after the launch): every shard CTA stores its output rows
    into EVERY rank's full y -- peer memory mapped over NVLink through CUDA
    IPC -- and publishes them on every rank's exchange words
    (rsp_stack_spec.xrank).  A dependent group on any rank starts once all
    ranks' CTAs of the previous group have published.

    ``layers``: this rank's shards (shard_rank = rank, shard_count = world);
    ``xs[i]``: a device tensor, or an int j = "the full output of linear j"
    (its copy in this rank's exchange area, assembled by all ranks);
    ``wait_prev`` as for :class:`layer.Stack`.  Every rank builds the same
    stack; the plans are checked to agree.  ``ipc`` / ``create`` exist for the
    CPU tests of the host logic."""

    def __init__(self, layers: Sequence[DecomposedLayer], xs, wait_prev=None, group=None,
                 device: int = 0, ipc: Optional[IpcOps] = None, create: bool = True):
        from . import _lib as L
        self.rank, self.world = _group_info(group)
        self.group = group
        self.layers = list(layers)
        self.ipc = ipc or IpcOps()
        m_full = [l.m_out for l in self.layers]
        rows = [(l.row_begin, l.row_end) for l in self.layers]
        for l, (rb, re) in zip(self.layers, rows):
            if (rb, re) != shard_rows(l.m_out, self.rank, self.world):
                raise ValueError("PeerStack: layers must be this rank's row shards")
        self.y_offs, self.xoff, self.nbytes = exchange_layout(m_full)
        self.base = self.ipc.alloc(device, self.nbytes)  # zeroed: y and the exchange words
        handles = _all_gather_object(self.ipc.export(self.base), group)
        self.bases = [self.base if p == self.rank else self.ipc.open(device, handles[p])
                      for p in range(self.world)]
        self.y_peers, self.xctr = exchange_tables(self.bases, self.y_offs, self.xoff, [r[0] for r in rows])
        self.y_devs = [self.base + off + 4 * rb for off, (rb, _) in zip(self.y_offs, rows)]
        self.x_devs = [self.base + self.y_offs[x] if isinstance(x, int) else x.data_ptr() for x in xs]
        self._h = None
        if not create:
            return
        self._keep = xs
        n = len(self.layers)
        sp = L.StackSpec()
        hp = (L.ct.c_void_p * n)(*[l.handle.value for l in self.layers])
        xp = (L.ct.c_void_p * n)(*self.x_devs)
        yp = (L.ct.c_void_p * n)(*self.y_devs)
        dts = {x.dtype for x in xs if not isinstance(x, int)} | ({torch.float32} if any(
            isinstance(x, int) for x in xs) else set())
        if len(dts) != 1 or not dts <= {torch.float32, torch.bfloat16}:
            # one activation dtype per stack; the exchange area holds fp32 outputs
            raise ValueError(f"PeerStack: all inputs must share one dtype (fp32 or bf16), got {dts}")
        sp.layers, sp.count, sp.x_devs, sp.y_devs = hp, n, xp, yp
        sp.x_dtype = L.RSP_BF16 if dts == {torch.bfloat16} else L.RSP_F32
        wp = None
        if wait_prev is not None:
            wp = (L.ct.c_uint8 * n)(*[1 if w else 0 for w in wait_prev])
            sp.wait_prev = L.ct.cast(wp, L.ct.POINTER(L.ct.c_uint8))
        sp.npeer = self.world
        flat = [p for pl in self.y_peers for p in pl]
        sp.y_peers = (L.ct.c_void_p * len(flat))(*flat)
        sp.xrank, sp.xself = self.world, self.rank
        sp.xctr = (L.ct.c_void_p * self.world)(*self.xctr)
        h = L.ct.c_void_p()
        torch.cuda.synchronize(device)
        L.check(L.lib().rsp_stack_create_spec(L.ct.byref(sp), L.ct.byref(h)), "rsp_stack_create_spec")
        self._h = h
        grids = (L.ct.c_uint32 * n)()
        L.check(L.lib().rsp_stack_grids(h, grids, n), "rsp_stack_grids")
        plans_agree(list(grids), group)

    def full_y(self, i: int):
        """Linear i's full output in this rank's exchange area (fp32 view;
        valid until :meth:`close`, which frees the area)."""
        return torch.as_tensor(_CudaArray(self.base + self.y_offs[i], self.layers[i].m_out, "<f4"),
                               device=f"cuda:{torch.cuda.current_device()}")

    def launch(self, stream=None) -> None:
        from . import _lib as L
        from .layer import _stream_ptr
        L.check(L.lib().rsp_stack_launch(self._h, _stream_ptr(stream)), "rsp_stack_launch")

    def close(self) -> None:
        from . import _lib as L
        if self._h:
            L.lib().rsp_stack_destroy(self._h)
            self._h = None
        for p, b in enumerate(getattr(self, "bases", [])):
            if p != self.rank:
                self.ipc.close(b)
        self.bases = []
        if getattr(self, "base", None):
            self.ipc.free(self.base)
            self.base = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
