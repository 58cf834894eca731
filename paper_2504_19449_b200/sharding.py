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
    captured into one CUDA graph when the runtime allows a graph launch
    inside a capture, else replayed eagerly.  Needs even shards (every
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
            st.launch(self.stream)
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
