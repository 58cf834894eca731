"""Host-side mirror of the reference operator API, over the C ABI.

Names, argument meaning and error behaviour follow the reference's
``namespace rsparse`` (core/include/rsparse/layer.hpp, sparsity.hpp,
matrix.hpp, search.hpp) so code written against the reference reads the
same here:

    reference (C++)                                  here
    ------------------------------------------------ -------------------------------
    SparsityPlan{keep_fraction, rank} sparsity.hpp:34 SparsityPlan
    DecomposedLayer               layer.hpp:38-48     DecomposedLayer
    forward(layer, x)             layer.hpp:75        forward / DecomposedLayer.forward
    gather_matvec(w_cols,x,kept)  layer.hpp:69-71     gather_matvec
    io_cost(layer)                layer.hpp:77        io_cost / DecomposedLayer.io_cost
    threshold_sparsify(x, s)      sparsity.hpp:43-44  threshold_sparsify
    top_k_by_magnitude(x, k)      matrix.hpp:63       top_k_by_magnitude
    Recipe::plan_for / rank_for   search.hpp:17-27    Recipe

Device memory and streams are PyTorch's (plumbing only): activations are
CUDA tensors, outputs are fp32 CUDA tensors.  All compute happens in
librsparse_b200.so; nothing here computes a result on the CPU.
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import check

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None


@dataclass
class SparsityPlan:
    """Per-layer knobs (sparsity.hpp:34-39): fraction of input channels kept
    exactly, and the rank routed through the low-rank factors."""
    keep_fraction: float = 1.0
    rank: int = 0


@dataclass
class IoReport:
    """io_cost (layer.hpp:51-55) plus the kernel's actual byte counts."""
    dense_bytes: int
    touched_bytes: int
    relative_cost: float
    kernel_weight_bytes: int
    kernel_total_bytes: int
    dense_weight_bytes: int


def _stream_ptr(stream=None) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def _x_dtype(x) -> int:
    if x.dtype == torch.float32:
        return L.RSP_F32
    if x.dtype == torch.bfloat16:
        return L.RSP_BF16
    raise L.UsageError(L.RSP_E_USAGE, f"activation dtype {x.dtype} unsupported (float32/bfloat16)")


def _src(a, name: str):
    """(pointer, dtype code, memory code, keepalive) for a weight source."""
    if torch is not None and isinstance(a, torch.Tensor):
        a = a.contiguous()
        code = {torch.float64: L.RSP_F64, torch.float32: L.RSP_F32, torch.bfloat16: L.RSP_BF16}.get(a.dtype)
        if code is None:
            raise L.UsageError(L.RSP_E_USAGE, f"{name}: dtype {a.dtype} unsupported")
        mem = L.RSP_MEM_DEVICE if a.is_cuda else L.RSP_MEM_HOST
        return a.data_ptr(), code, mem, a
    arr = np.ascontiguousarray(a)
    if arr.dtype == np.float64:
        code = L.RSP_F64
    elif arr.dtype == np.float32:
        code = L.RSP_F32
    else:
        arr = arr.astype(np.float64)
        code = L.RSP_F64
    return arr.ctypes.data, code, L.RSP_MEM_HOST, arr


class DecomposedLayer:
    """A B200-resident rsparse::DecomposedLayer.

    ``w`` is the m_out x m_in weight (``w_layout="row"``, rsparse::Matrix) or
    the reference's column-major ``w_cols`` data as an (m_in, m_out) array
    (``w_layout="col"``).  ``a_r`` (m_out x r) = U_r sqrt(Sigma_r) and ``b_r``
    (r x m_in) = sqrt(Sigma_r) Vt_r are the precomputed factors
    (layer.cpp:61-66).  Sources may be numpy arrays or torch tensors (host or
    CUDA; f64/f32/bf16).  ``weight_dtype`` is the HBM storage type.
    """

    def __init__(self, w, a_r=None, b_r=None, plan: Optional[SparsityPlan] = None, *,
                 keep_fraction: Optional[float] = None, rank: Optional[int] = None,
                 weight_dtype: str = "bf16", w_layout: str = "row", k: Optional[int] = None,
                 device: int = 0, shard_rank: int = 0, shard_count: int = 1,
                 deterministic: bool = False, batch_tcgen05: bool = False):
        if plan is None:
            plan = SparsityPlan(1.0 if keep_fraction is None else keep_fraction,
                                0 if rank is None else rank)
        self.plan = plan
        shape = tuple(w.shape)
        if w_layout == "row":
            m_out, m_in = shape
        elif w_layout == "col":
            m_in, m_out = shape
        else:
            raise L.UsageError(L.RSP_E_USAGE, "w_layout must be 'row' or 'col'")
        r = int(plan.rank)
        wp, wdt, wmem, wk = _src(w, "w")
        keep = [wk]
        ap = bp = 0
        if r > 0:
            if a_r is None or b_r is None:
                raise L.UsageError(L.RSP_E_USAGE, "rank > 0 needs a_r and b_r")
            if tuple(a_r.shape) != (m_out, r) or tuple(b_r.shape) != (r, m_in):
                raise L.UsageError(L.RSP_E_USAGE, f"factor shapes {tuple(a_r.shape)} / {tuple(b_r.shape)} "
                                   f"do not match m_out={m_out}, m_in={m_in}, r={r}")
            ap, adt, amem, ak = _src(a_r, "a_r")
            bp, bdt, bmem, bk = _src(b_r, "b_r")
            if not (adt == bdt == wdt and amem == bmem == wmem):
                raise L.UsageError(L.RSP_E_USAGE, "w, a_r and b_r must share dtype and memory")
            keep += [ak, bk]
        d = L.LinearDesc()
        d.m_in, d.m_out, d.rank = m_in, m_out, r
        d.keep_fraction = float(plan.keep_fraction)
        d.k_override = -1 if k is None else int(k)
        d.weight_dtype = {"bf16": L.RSP_BF16, "f32": L.RSP_F32, "fp32": L.RSP_F32}[weight_dtype]
        d.src_dtype, d.src_memory = wdt, wmem
        d.w_layout = L.RSP_W_ROW_MAJOR if w_layout == "row" else L.RSP_W_COL_MAJOR
        d.w, d.a_r, d.b_r = wp, ap, bp
        d.device, d.shard_rank, d.shard_count = device, shard_rank, shard_count
        d.flags = (L.RSP_FLAG_DETERMINISTIC if deterministic else 0) | \
            (L.RSP_FLAG_BATCH_TCGEN05 if batch_tcgen05 else 0)
        h = ct.c_void_p()
        if torch is not None and wmem == L.RSP_MEM_DEVICE:
            torch.cuda.synchronize(device)
        check(L.lib().rsp_linear_create(ct.byref(d), ct.byref(h)), "rsp_linear_create")
        self._adopt(h, device, weight_dtype)

    def _adopt(self, h, device: int, weight_dtype: str) -> None:
        self._h = h
        self.device = device
        self.weight_dtype = weight_dtype
        info = L.LinearInfo()
        check(L.lib().rsp_linear_info_get(self._h, ct.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in L.LinearInfo._fields_}
        self.m_in, self.m_out = info.m_in, info.m_out
        self.k = info.k
        self.row_begin, self.row_end = info.row_begin, info.row_end
        self._ws = None

    # -- RSPL files (layer.cpp:243-301) ---------------------------------------
    @classmethod
    def load_rspl(cls, path: str, *, weight_dtype: str = "f32", k: Optional[int] = None,
                  device: int = 0, shard_rank: int = 0, shard_count: int = 1,
                  deterministic: bool = False) -> "DecomposedLayer":
        """read_decomposed_layer (layer.hpp:95) straight into HBM."""
        hdr = read_rspl_header(path)
        d = L.LinearDesc()
        d.k_override = -1 if k is None else int(k)
        d.weight_dtype = {"bf16": L.RSP_BF16, "f32": L.RSP_F32, "fp32": L.RSP_F32}[weight_dtype]
        d.device, d.shard_rank, d.shard_count = device, shard_rank, shard_count
        d.flags = L.RSP_FLAG_DETERMINISTIC if deterministic else 0
        h = ct.c_void_p()
        check(L.lib().rsp_linear_load_rspl(path.encode(), ct.byref(d), ct.byref(h)), "rsp_linear_load_rspl")
        self = cls.__new__(cls)
        self.plan = SparsityPlan(hdr["keep_fraction"], hdr["rank"])
        self._adopt(h, device, weight_dtype)
        return self

    def save_rspl(self, path: str) -> None:
        """write_decomposed_layer (layer.hpp:93) of the device-resident values."""
        check(L.lib().rsp_linear_save_rspl(self._h, path.encode()), "rsp_linear_save_rspl")

    @property
    def selected_components(self) -> List[int]:
        r = int(self.plan.rank)
        buf = (ct.c_uint32 * max(r, 1))()
        check(L.lib().rsp_linear_components(self._h, buf), "rsp_linear_components")
        return list(buf)[:r]

    # -- plumbing ------------------------------------------------------------
    @property
    def handle(self) -> ct.c_void_p:
        return self._h

    def workspace_size(self) -> int:
        return int(L.lib().rsp_linear_workspace_size(self._h, 1))

    def workspace(self):
        """A zero-initialised per-layer workspace (torch uint8 CUDA tensor)."""
        if self._ws is None:
            self._ws = torch.zeros(self.workspace_size(), dtype=torch.uint8, device=f"cuda:{self.device}")
        return self._ws

    def close(self) -> None:
        if getattr(self, "_h", None):
            L.lib().rsp_linear_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- operator --------------------------------------------------------------
    def forward(self, x, out=None, workspace=None, stream=None):
        """rsparse::forward(layer, x) (layer.cpp:95-123) for one token, or a
        (batch, m_in) tensor of tokens run as independent forwards.  Returns
        fp32 (m_shard,) or (batch, m_shard) on the layer's device."""
        if x.shape[-1] != self.m_in:  # layer.cpp:96-99
            raise L.UsageError(L.RSP_E_USAGE, f"forward: input length {x.shape[-1]} does not match m_in {self.m_in}")
        x = x.contiguous()
        batch = 1 if x.dim() == 1 else x.shape[0]
        m = self.row_end - self.row_begin
        if out is None:
            out = torch.empty((m,) if x.dim() == 1 else (batch, m), dtype=torch.float32, device=x.device)
        ws = self.workspace() if workspace is None else workspace
        check(L.lib().rsp_linear_forward(self._h, x.data_ptr(), _x_dtype(x), out.data_ptr(), batch,
                                         ws.data_ptr(), ws.numel(), _stream_ptr(stream)),
              "rsp_linear_forward")
        return out

    __call__ = forward

    def dense_forward(self, x, out=None, workspace=None, stream=None):
        """Dense baseline of the same layer: all m_in channels through W."""
        x = x.contiguous()
        m = self.row_end - self.row_begin
        if out is None:
            out = torch.empty(m, dtype=torch.float32, device=x.device)
        ws = self.workspace() if workspace is None else workspace
        check(L.lib().rsp_linear_dense_forward(self._h, x.data_ptr(), _x_dtype(x), out.data_ptr(),
                                               ws.data_ptr(), ws.numel(), _stream_ptr(stream)),
              "rsp_linear_dense_forward")
        return out

    def forward_host(self, x: np.ndarray, x_dtype: str = "f32") -> np.ndarray:
        """End-to-end path with host buffers: H2D, fused forward, D2H.
        Returns float64 like the reference's std::vector<double>."""
        if x_dtype == "bf16":
            xt = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16)
            xa = xt.view(torch.int16).numpy()
            code = L.RSP_BF16
        else:
            xa = np.ascontiguousarray(x, dtype=np.float32)
            code = L.RSP_F32
        if xa.shape[-1] != self.m_in:
            raise L.UsageError(L.RSP_E_USAGE, f"forward: input length {xa.shape[-1]} does not match m_in {self.m_in}")
        batch = 1 if xa.ndim == 1 else xa.shape[0]
        m = self.row_end - self.row_begin
        y = np.empty((m,) if xa.ndim == 1 else (batch, m), dtype=np.float64)
        check(L.lib().rsp_linear_forward_host(self._h, xa.ctypes.data, code, y.ctypes.data, L.RSP_F64, batch),
              "rsp_linear_forward_host")
        return y

    def selected(self, x) -> np.ndarray:
        """The channel set S the forward keeps for x (ascending)."""
        S = np.empty(max(self.k, 1), dtype=np.int32)
        kk = ct.c_uint32()
        check(L.lib().rsp_linear_selected(self._h, x.contiguous().data_ptr(), _x_dtype(x),
                                          S.ctypes.data_as(ct.POINTER(ct.c_int32)), ct.byref(kk)),
              "rsp_linear_selected")
        return S[: kk.value].astype(np.int64)

    def io_cost(self) -> IoReport:
        rep = L.IoReport()
        check(L.lib().rsp_linear_io_cost(self._h, ct.byref(rep)))
        return IoReport(**{f: getattr(rep, f) for f, _ in L.IoReport._fields_})

    def export(self):
        """(W m_shard x m_in, a_r m_shard x r, b_r r x m_in) as float64: exactly the
        values the kernels read (after dtype rounding)."""
        m, n, r = self.row_end - self.row_begin, self.m_in, self.plan.rank
        outs = []
        for which, shape in ((0, (m, n)), (1, (m, r)), (2, (r, n))):
            a = np.zeros(shape, dtype=np.float64)
            if a.size:
                check(L.lib().rsp_linear_export(self._h, which, a.ctypes.data_as(ct.POINTER(ct.c_double))))
            outs.append(a)
        return tuple(outs)


def read_rspl_header(path: str) -> dict:
    """RSPL header fields (host-only parse; RSP_E_IO -> IoError like io_error)."""
    h = L.RsplHeader()
    check(L.lib().rsp_rspl_read(path.encode(), ct.byref(h), None, None, None, None), "rsp_rspl_read")
    return {f: getattr(h, f) for f, _ in L.RsplHeader._fields_}


def read_rspl(path: str) -> dict:
    """Host-only read of a whole RSPL file (read_decomposed_layer's fields as
    float32 arrays: w_cols (m_in, m_out), a_r (m_out, r), b_r (r, m_in), comps)."""
    hdr = read_rspl_header(path)
    n, m, r = hdr["m_in"], hdr["m_out"], hdr["rank"]
    w = np.empty((n, m), np.float32)
    a = np.empty((m, r), np.float32)
    b = np.empty((r, n), np.float32)
    c = np.empty(max(r, 1), np.uint32)
    check(L.lib().rsp_rspl_read(path.encode(), ct.byref(L.RsplHeader()), w.ctypes.data, a.ctypes.data,
                                b.ctypes.data, c.ctypes.data), "rsp_rspl_read")
    return dict(hdr, w_cols=w, a_r=a, b_r=b, comps=c[:r])


def read_decomposed_layer(path: str, **kw) -> DecomposedLayer:
    """rsparse::read_decomposed_layer (layer.hpp:95), device-resident."""
    return DecomposedLayer.load_rspl(path, **kw)


def write_decomposed_layer(layer: DecomposedLayer, path: str) -> None:
    """rsparse::write_decomposed_layer (layer.hpp:93)."""
    layer.save_rspl(path)


def forward(layer: DecomposedLayer, x, **kw):
    """rsparse::forward (layer.hpp:75)."""
    return layer.forward(x, **kw)


def io_cost(layer: DecomposedLayer) -> IoReport:
    """rsparse::io_cost (layer.hpp:77)."""
    return layer.io_cost()


def gather_matvec(layer: DecomposedLayer, x, kept: Sequence[int], stream=None):
    """rsparse::gather_matvec(w_cols, x, kept, touched_bytes) (layer.hpp:69-71):
    y = sum over kept (in list order) of x_j * column j.  Returns (y, touched)."""
    if x.shape[-1] != layer.m_in:
        raise L.UsageError(L.RSP_E_USAGE, f"gather_matvec: input length {x.shape[-1]} does not match "
                           f"column count {layer.m_in}")
    kept = np.ascontiguousarray(np.asarray(kept, dtype=np.int64))
    y = torch.empty(layer.row_end - layer.row_begin, dtype=torch.float32, device=x.device)
    touched = ct.c_uint64(0)
    x = x.contiguous()
    check(L.lib().rsp_gather_matvec(layer.handle, x.data_ptr(), _x_dtype(x),
                                    kept.ctypes.data_as(ct.POINTER(ct.c_int64)), kept.size,
                                    y.data_ptr(), ct.byref(touched), _stream_ptr(stream)),
          "rsp_gather_matvec")
    return y, touched.value


def top_k_by_magnitude(x, k: int, with_rest: bool = False, stream=None):
    """rsparse::top_k_by_magnitude (matrix.cpp:100-117) on a CUDA vector:
    indices of the k largest |x|, ties to the lower index, ascending (int32)."""
    n = x.numel()
    x = x.contiguous()
    kept = torch.empty(max(k, 1), dtype=torch.int32, device=x.device)
    rest = torch.empty(max(n - k, 1), dtype=torch.int32, device=x.device) if with_rest else None
    check(L.lib().rsp_top_k_by_magnitude(x.data_ptr(), _x_dtype(x), n, k, kept.data_ptr(),
                                         rest.data_ptr() if rest is not None else None,
                                         _stream_ptr(stream)), "rsp_top_k_by_magnitude")
    kept = kept[:k]
    return (kept, rest[: n - k]) if with_rest else kept


def threshold_sparsify(x, keep_fraction: float, stream=None):
    """rsparse::threshold_sparsify (sparsity.cpp:20-32): (sparse_x fp32, kept int32)."""
    n = x.numel()
    x = x.contiguous()
    sx = torch.empty(n, dtype=torch.float32, device=x.device)
    kept = torch.empty(max(n, 1), dtype=torch.int32, device=x.device)
    kk = ct.c_uint32()
    check(L.lib().rsp_threshold_sparsify(x.data_ptr(), _x_dtype(x), n, float(keep_fraction),
                                         sx.data_ptr(), kept.data_ptr(), ct.byref(kk),
                                         _stream_ptr(stream)), "rsp_threshold_sparsify")
    return sx, kept[: kk.value]


def shard_rows(m_out: int, shard_rank: int, shard_count: int):
    """Output rows [begin, end) owned by one shard (the partition create() applies)."""
    b, e = ct.c_uint32(), ct.c_uint32()
    check(L.lib().rsp_shard_rows(m_out, shard_rank, shard_count, ct.byref(b), ct.byref(e)), "shard_rows")
    return b.value, e.value


def keep_count(keep_fraction: float, n: int) -> int:
    """k = ceil(s*n) (sparsity.cpp:26-27)."""
    k = ct.c_uint32()
    check(L.lib().rsp_keep_count(float(keep_fraction), int(n), ct.byref(k)), "keep_count")
    return k.value


class Recipe:
    """rsparse::Recipe (search.hpp:17-27): per-layer rho_i (sparse share of
    the I/O budget) and budget C_i."""

    def __init__(self, rho: Sequence[float], budget: Sequence[float]):
        if len(rho) != len(budget):
            raise L.UsageError(L.RSP_E_USAGE, "rho and budget lengths differ")
        self.rho = [float(v) for v in rho]
        self.budget = [float(v) for v in budget]

    def num_layers(self) -> int:
        return len(self.rho)

    def keep_fraction(self, i: int) -> float:
        return self.rho[i] * self.budget[i]

    def plan_for(self, i: int, m_in: int, m_out: int) -> SparsityPlan:
        s, r = ct.c_double(), ct.c_uint32()
        check(L.lib().rsp_plan_for(self.rho[i], self.budget[i], m_in, m_out, ct.byref(s), ct.byref(r)))
        return SparsityPlan(s.value, r.value)

    def rank_for(self, i: int, m_in: int, m_out: int) -> int:
        return self.plan_for(i, m_in, m_out).rank


class Stack:
    """A decode-order sequence of forwards run by one persistent kernel launch
    (captured once into a CUDA graph; rsp_stack_create_ex).

    ``wait_prev[i]`` (default all True) says linear i's input depends on
    linear i-1's output, so it starts only once that output is complete.
    Linears that share the previous linear's input (q/k/v, gate/up) pass False
    and overlap with it."""

    def __init__(self, layers: List[DecomposedLayer], xs, ys, dense: bool = False,
                 wait_prev: Optional[Sequence[bool]] = None, silu_gate: Optional[Sequence[bool]] = None,
                 y_peers: Optional[Sequence[Sequence]] = None, max_ctas: int = 0):
        """y_peers[i] (optional): the destinations of linear i's output rows --
        every rank's copy of the full y at this shard's first row (tensors or
        device pointers); the kernel writes all of them (rsp_stack_create_spec)."""
        self.layers = layers
        self.xs, self.ys = xs, ys
        n = len(layers)
        if len({x.dtype for x in xs}) != 1:  # the ABI takes one activation dtype per stack
            raise L.UsageError(L.RSP_E_USAGE, "stack inputs must share one dtype")
        hp = (ct.c_void_p * n)(*[l.handle.value for l in layers])
        xp = (ct.c_void_p * n)(*[x.data_ptr() for x in xs])
        yp = (ct.c_void_p * n)(*[y.data_ptr() for y in ys])
        wp = None
        if wait_prev is not None:
            if len(wait_prev) != n:
                raise L.UsageError(L.RSP_E_USAGE, "wait_prev length differs from the layer count")
            wp = (ct.c_uint8 * n)(*[1 if w else 0 for w in wait_prev])
        ops = None
        if silu_gate is not None:
            # RSP_XOP_SILU_GATE: xs[i] holds [a | g] (fp32, 2 m_in); the input is a * silu(g)
            if len(silu_gate) != n:
                raise L.UsageError(L.RSP_E_USAGE, "silu_gate length differs from the layer count")
            ops = (ct.c_uint8 * n)(*[L.RSP_XOP_SILU_GATE if g else L.RSP_XOP_NONE for g in silu_gate])
        h = ct.c_void_p()
        torch.cuda.synchronize()
        if y_peers is None and not max_ctas:
            check(L.lib().rsp_stack_create_ops(hp, n, xp, _x_dtype(xs[0]), yp, 1 if dense else 0, wp, ops,
                                               ct.byref(h)), "rsp_stack_create_ops")
        else:
            npeer = len(y_peers[0]) if y_peers is not None else 1
            if y_peers is not None and (len(y_peers) != n or any(len(p) != npeer for p in y_peers)):
                raise L.UsageError(L.RSP_E_USAGE, "y_peers needs the same number of destinations for every linear")
            ptrs = [(t.data_ptr() if hasattr(t, "data_ptr") else int(t)) for pl in (y_peers or []) for t in pl]
            self._peers = y_peers
            sp = L.StackSpec()
            sp.max_ctas = int(max_ctas)
            sp.layers, sp.count, sp.x_devs, sp.x_dtype, sp.y_devs = hp, n, xp, _x_dtype(xs[0]), yp
            sp.dense = 1 if dense else 0
            sp.wait_prev = ct.cast(wp, ct.POINTER(ct.c_uint8)) if wp is not None else None
            sp.x_ops = ct.cast(ops, ct.POINTER(ct.c_uint8)) if ops is not None else None
            sp.npeer = npeer
            sp.y_peers = (ct.c_void_p * len(ptrs))(*ptrs) if ptrs else None
            check(L.lib().rsp_stack_create_spec(ct.byref(sp), ct.byref(h)), "rsp_stack_create_spec")
        self._h = h

    def launch(self, stream=None, direct: bool = False) -> None:
        """One token through the stack.  ``direct``: a plain kernel launch
        instead of the stack's CUDA graph (capturable into a caller's graph)."""
        if direct:
            check(L.lib().rsp_stack_launch_direct(self._h, _stream_ptr(stream)), "rsp_stack_launch_direct")
        else:
            check(L.lib().rsp_stack_launch(self._h, _stream_ptr(stream)), "rsp_stack_launch")

    def info(self):
        return {"handle": self._h.value}

    def io_spans(self):
        """(x_bytes, y_bytes): the device spans covering all inputs / outputs."""
        xb, yb = ct.c_size_t(), ct.c_size_t()
        check(L.lib().rsp_stack_io_spans(self._h, ct.byref(xb), ct.byref(yb)), "rsp_stack_io_spans")
        return xb.value, yb.value

    def launch_host(self, x_host, y_host, stream=None) -> None:
        """End to end through the ABI (rsp_stack_launch_host): H2D of x_host
        (a host tensor / array covering the stack's input span), the stack,
        D2H of the output span into y_host; returns synchronised."""
        xb, yb = self.io_spans()
        xp = x_host.data_ptr() if hasattr(x_host, "data_ptr") else x_host.ctypes.data
        yp = y_host.data_ptr() if hasattr(y_host, "data_ptr") else y_host.ctypes.data
        check(L.lib().rsp_stack_launch_host(self._h, xp, xb, yp, yb, _stream_ptr(stream)), "rsp_stack_launch_host")

    def close(self) -> None:
        if getattr(self, "_h", None):
            L.lib().rsp_stack_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TokenParallelStack:
    """A decode stack over a small batch of B tokens as B independent
    persistent stack launches on disjoint SM partitions (max_ctas = SMs / B),
    forked onto B streams and joined -- captured into one CUDA graph.  The
    reference semantics of a batch (B independent forward
    calls) taken literally: each token keeps its own selection; the
    per-dependency-step fixed costs of the B tokens overlap instead of adding
    up.  xs[i] / ys[i] are (B, m_in) / (B, m_out) per linear."""

    def __init__(self, layers: List[DecomposedLayer], xs, ys, wait_prev: Optional[Sequence[bool]] = None,
                 stream=None):
        self.B = int(xs[0].shape[0])
        dev = xs[0].device
        sms = int(L.lib().rsp_device_sm_count(dev.index or 0))
        self.stacks = [Stack(layers, [x[b] for x in xs], [y[b] for y in ys], wait_prev=wait_prev,
                             max_ctas=max(1, sms // self.B)) for b in range(self.B)]
        self.stream = stream or torch.cuda.current_stream(dev)
        self.side = [torch.cuda.Stream(device=dev) for _ in range(self.B)]
        # fork / B plain stack launches (rsp_stack_launch_direct) / join,
        # captured once into one CUDA graph on a private stream
        with torch.cuda.stream(self.stream):
            self._run(self.stream)
            torch.cuda.synchronize()
        cap = torch.cuda.Stream(device=dev)
        cap.wait_stream(self.stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            self._run(cap)
        self.graph = g

    def _run(self, root):
        fork = torch.cuda.Event()
        fork.record(root)
        joins = []
        for st, sd in zip(self.stacks, self.side):
            sd.wait_event(fork)
            st.launch(sd, direct=True)
            ev = torch.cuda.Event()
            ev.record(sd)
            joins.append(ev)
        for ev in joins:
            root.wait_event(ev)

    def launch(self, stream=None) -> None:
        with torch.cuda.stream(stream or self.stream):
            self.graph.replay()

    def close(self) -> None:
        for st in self.stacks:
            st.close()



class BatchedStack:
    """A decode stack over a batch of B tokens (xs[i]: (B, m_in), ys[i]:
    (B, m_out)) with the executor chosen by B (profiles/r02_config3_*):

    * B == 1: the persistent stack kernel (:class:`Stack`);
    * 2 <= B <= TOKEN_PARALLEL_MAX: B concurrent per-token stacks on disjoint
      SM partitions (:class:`TokenParallelStack`);
    * larger B: the union-of-masks pass per linear (rsp_linear_forward with
      batch = B: each W row of the tokens' union read once), captured into one
      CUDA graph.

    Every token keeps its own selection (the reference's batch semantics,
    SPEC.md:325, 331)."""

    TOKEN_PARALLEL_MAX = 5  # measured crossover: B = 5 1.33 vs 1.39 ms, B = 6 1.25 vs 1.17 (token-parallel vs union)

    def __init__(self, layers: List[DecomposedLayer], xs, ys, wait_prev: Optional[Sequence[bool]] = None,
                 stream=None):
        self.B = int(xs[0].shape[0])
        self.stream = stream or torch.cuda.current_stream(xs[0].device)
        self.graph = None
        if self.B == 1:
            self.mode = "persistent"
            self.impl = Stack(layers, [x[0] for x in xs], [y[0] for y in ys], wait_prev=wait_prev)
        elif self.B <= self.TOKEN_PARALLEL_MAX:
            self.mode = "token_parallel"
            self.impl = TokenParallelStack(layers, xs, ys, wait_prev=wait_prev, stream=self.stream)
        else:
            self.mode = "union_per_linear"
            self.impl = None
            self.layers, self.xs, self.ys = layers, xs, ys
            self.ws = [l.workspace() for l in layers]
            # captured on a private stream (a capture cannot run on the
            # legacy default stream), replayed on self.stream
            cap = torch.cuda.Stream(device=xs[0].device)
            cap.wait_stream(self.stream)
            self._run(cap)
            cap.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cap):
                self._run(cap)
            self.graph = g

    def _run(self, stream):
        for l, x, y, ws in zip(self.layers, self.xs, self.ys, self.ws):
            l.forward(x, out=y, workspace=ws, stream=stream)

    def launch(self, stream=None) -> None:
        if self.graph is not None:
            with torch.cuda.stream(stream or self.stream):
                self.graph.replay()
        elif self.mode == "persistent":
            self.impl.launch(stream or self.stream)
        else:
            self.impl.launch()

    def close(self) -> None:
        if self.impl is not None:
            self.impl.close()
