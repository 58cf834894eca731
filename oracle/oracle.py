"""ctypes access to the parity checkers.  TEST INFRASTRUCTURE ONLY.

Two libraries, one Python surface:

* ``C``   -- oracle/librsparse_oracle.so, the plain-C restatement of the
             reference hot path (oracle/rsparse_oracle.c).
* ``REF`` -- oracle/_ref/librsparse_ref.so, the unmodified reference sources
             compiled in place plus oracle/ref_shim.cpp (absent when the
             reference tree was not available at build time).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module.  The product (paper_2504_19449_b200) never does.
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
C_PATH = os.path.join(HERE, "librsparse_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "librsparse_ref.so")

_dp = ct.POINTER(ct.c_double)
_i64p = ct.POINTER(ct.c_int64)
_u64p = ct.POINTER(ct.c_uint64)
_szp = ct.POINTER(ct.c_size_t)


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: status {status}")
        self.status = status


class UsageError(OracleError):
    pass


def _raise(st: int, what: str):
    if st == 0:
        return
    if st == 2:
        raise UsageError(st, what)
    raise OracleError(st, what)


def build(quiet: bool = True) -> None:
    """Compile the oracle (and the reference shim when /root/reference exists)."""
    out = subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")],
                         capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _as_f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class _Lib:
    """Common wrapper.  ``prefix`` is "rspo" (C restatement) or "rspr" (reference)."""

    def __init__(self, path: str, prefix: str):
        self.path = path
        self.prefix = prefix
        self.lib = ct.CDLL(path)
        L, p = self.lib, prefix
        self._fill_normal = getattr(L, f"{p}_fill_normal")
        self._fill_normal.argtypes = [ct.c_uint64, ct.c_double, ct.c_double, _dp, ct.c_size_t]
        self._fill_normal.restype = None
        self._fill_u = getattr(L, f"{p}_fill_uniform01")
        self._fill_u.argtypes = [ct.c_uint64, _dp, ct.c_size_t]
        self._fill_u.restype = None
        self._derive = getattr(L, f"{p}_derive_seed")
        self._derive.argtypes = [ct.c_uint64, ct.c_char_p]
        self._derive.restype = ct.c_uint64
        self._topk = getattr(L, f"{p}_top_k_by_magnitude")
        self._topk.argtypes = [_dp, ct.c_size_t, ct.c_size_t, _i64p]
        self._topk.restype = ct.c_int
        self._thr = getattr(L, f"{p}_threshold_sparsify")
        self._thr.argtypes = [_dp, ct.c_size_t, ct.c_double, _dp, _i64p, _szp]
        self._thr.restype = ct.c_int
        self._gmv = getattr(L, f"{p}_gather_matvec")
        self._gmv.argtypes = [_dp, ct.c_size_t, ct.c_size_t, _dp, _i64p, ct.c_size_t, _dp, _u64p]
        self._gmv.restype = ct.c_int
        self._io = getattr(L, f"{p}_io_cost")
        self._io.argtypes = [ct.c_size_t, ct.c_size_t, ct.c_double, ct.c_size_t, _u64p, _u64p,
                             ct.POINTER(ct.c_double)]
        self._io.restype = None

    # -- rng.hpp -----------------------------------------------------------
    def derive_seed(self, root: int, tag: str) -> int:
        return int(self._derive(root, tag.encode()))

    def normal(self, seed: int, count: int, mean: float = 0.0, std: float = 1.0) -> np.ndarray:
        out = np.empty(count, dtype=np.float64)
        self._fill_normal(seed, mean, std, _d(out), count)
        return out

    def uniform01(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.float64)
        self._fill_u(seed, _d(out), count)
        return out

    # -- matrix.cpp / sparsity.cpp ---------------------------------------
    def top_k_by_magnitude(self, x, k: int) -> np.ndarray:
        x = _as_f64(x)
        out = np.empty(max(k, 1), dtype=np.int64)
        _raise(self._topk(_d(x), x.size, k, out.ctypes.data_as(_i64p)), "top_k_by_magnitude")
        return out[:k].copy()

    def threshold_sparsify(self, x, keep_fraction: float):
        x = _as_f64(x)
        n = x.size
        sx = np.empty(max(n, 1), dtype=np.float64)
        kept = np.empty(max(n, 1), dtype=np.int64)
        k = ct.c_size_t(0)
        _raise(self._thr(_d(x), n, keep_fraction, _d(sx), kept.ctypes.data_as(_i64p), ct.byref(k)),
               "threshold_sparsify")
        return sx[:n].copy(), kept[: k.value].copy()

    # -- layer.cpp ---------------------------------------------------------
    def gather_matvec(self, w_cols, x, kept, count_bytes: bool = False):
        """``w_cols`` is the reference ColMajorMatrix data as an (n, m) array
        (row j == column j of W)."""
        w_cols = _as_f64(w_cols)
        n, m = w_cols.shape
        x = _as_f64(x)
        kept = np.ascontiguousarray(np.asarray(kept, dtype=np.int64))
        y = np.empty(max(m, 1), dtype=np.float64)
        tb = ct.c_uint64(0)
        _raise(self._gmv(_d(w_cols), m, n, _d(x), kept.ctypes.data_as(_i64p), kept.size, _d(y),
                         ct.byref(tb)), "gather_matvec")
        return (y[:m].copy(), tb.value) if count_bytes else y[:m].copy()

    def io_cost(self, m_in: int, m_out: int, keep_fraction: float, rank: int):
        d, t, rc = ct.c_uint64(), ct.c_uint64(), ct.c_double()
        self._io(m_in, m_out, keep_fraction, rank, ct.byref(d), ct.byref(t), ct.byref(rc))
        return {"dense_bytes": d.value, "touched_bytes": t.value, "relative_cost": rc.value}


class COracle(_Lib):
    """The C restatement (oracle/rsparse_oracle.c)."""

    class _Layer(ct.Structure):
        _fields_ = [("m_in", ct.c_size_t), ("m_out", ct.c_size_t), ("rank", ct.c_size_t),
                    ("keep_fraction", ct.c_double), ("w_cols", _dp), ("a_r", _dp), ("b_r", _dp)]

    def __init__(self, path: str = C_PATH):
        super().__init__(path, "rspo")
        L = self.lib
        L.rspo_forward_ex.argtypes = [ct.POINTER(self._Layer), _dp, _dp, _i64p, _szp]
        L.rspo_forward_ex.restype = ct.c_int
        L.rspo_forward_many.argtypes = [ct.POINTER(self._Layer), ct.POINTER(_dp), ct.POINTER(_dp),
                                        ct.c_size_t, ct.c_int]
        L.rspo_forward_many.restype = ct.c_int
        L.rspo_matvec.argtypes = [_dp, ct.c_size_t, ct.c_size_t, _dp, _dp]
        L.rspo_matvec.restype = None
        L.rspo_rank_for.argtypes = [ct.c_double, ct.c_double, ct.c_size_t, ct.c_size_t]
        L.rspo_rank_for.restype = ct.c_size_t
        L.rspo_keep_count.argtypes = [ct.c_double, ct.c_size_t]
        L.rspo_keep_count.restype = ct.c_size_t

    def make_layer(self, w_cols, a_r, b_r, keep_fraction: float):
        """Returns (struct, keepalive).  w_cols (n, m); a_r (m, r); b_r (r, n)."""
        w_cols, a_r, b_r = _as_f64(w_cols), _as_f64(a_r), _as_f64(b_r)
        n, m = w_cols.shape
        r = a_r.shape[1] if a_r.ndim == 2 else 0
        s = self._Layer(n, m, r, keep_fraction, _d(w_cols), _d(a_r), _d(b_r))
        return s, (w_cols, a_r, b_r)

    def forward(self, w_cols, a_r, b_r, keep_fraction: float, x, return_kept: bool = False):
        layer, keep = self.make_layer(w_cols, a_r, b_r, keep_fraction)
        x = _as_f64(x)
        if x.size != layer.m_in:
            raise UsageError(2, "forward: input length mismatch")
        y = np.empty(max(layer.m_out, 1), dtype=np.float64)
        kept = np.empty(max(layer.m_in, 1), dtype=np.int64)
        k = ct.c_size_t(0)
        _raise(self.lib.rspo_forward_ex(ct.byref(layer), _d(x), _d(y),
                                        kept.ctypes.data_as(_i64p), ct.byref(k)), "forward")
        y = y[: layer.m_out].copy()
        return (y, kept[: k.value].copy()) if return_kept else y

    def forward_many(self, layers, xs, threads: int = 1):
        """layers: list of (w_cols, a_r, b_r, s); xs: list of vectors.  Returns ys."""
        structs, keep = [], []
        for (w, a, b, s) in layers:
            st, kk = self.make_layer(w, a, b, s)
            structs.append(st)
            keep.append(kk)
        arr = (self._Layer * len(structs))(*structs)
        xs = [_as_f64(x) for x in xs]
        ys = [np.empty(st.m_out, dtype=np.float64) for st in structs]
        xp = (_dp * len(xs))(*[_d(x) for x in xs])
        yp = (_dp * len(ys))(*[_d(y) for y in ys])
        _raise(self.lib.rspo_forward_many(arr, xp, yp, len(structs), threads), "forward_many")
        return ys

    def matvec(self, w, x):
        w, x = _as_f64(w), _as_f64(x)
        y = np.empty(w.shape[0], dtype=np.float64)
        self.lib.rspo_matvec(_d(w), w.shape[0], w.shape[1], _d(x), _d(y))
        return y

    def rank_for(self, rho: float, budget: float, m_in: int, m_out: int) -> int:
        return int(self.lib.rspo_rank_for(rho, budget, m_in, m_out))

    def plan_for(self, rho: float, budget: float, m_in: int, m_out: int):
        return rho * budget, self.rank_for(rho, budget, m_in, m_out)

    def keep_count(self, keep_fraction: float, n: int) -> int:
        return int(self.lib.rspo_keep_count(keep_fraction, n))


class RefOracle(_Lib):
    """The reference library itself (oracle/_ref/librsparse_ref.so)."""

    def __init__(self, path: str = REF_PATH):
        super().__init__(path, "rspr")
        L = self.lib
        L.rspr_layer_create.argtypes = [ct.c_size_t, ct.c_size_t, ct.c_size_t, ct.c_double, _dp,
                                        _dp, _dp]
        L.rspr_layer_create.restype = ct.c_void_p
        L.rspr_layer_destroy.argtypes = [ct.c_void_p]
        L.rspr_layer_destroy.restype = None
        L.rspr_layer_forward.argtypes = [ct.c_void_p, _dp, _dp]
        L.rspr_layer_forward.restype = ct.c_int
        L.rspr_forward_many.argtypes = [ct.POINTER(ct.c_void_p), ct.POINTER(_dp), ct.POINTER(_dp),
                                        ct.c_size_t, ct.c_int]
        L.rspr_forward_many.restype = ct.c_int
        L.rspr_matvec.argtypes = [_dp, ct.c_size_t, ct.c_size_t, _dp, _dp]
        L.rspr_matvec.restype = ct.c_int
        L.rspr_plan_for.argtypes = [ct.c_double, ct.c_double, ct.c_size_t, ct.c_size_t,
                                    ct.POINTER(ct.c_double), _szp]
        L.rspr_plan_for.restype = None
        L.rspr_decompose_uniform.argtypes = [_dp, ct.c_size_t, ct.c_size_t, ct.c_double,
                                             ct.c_size_t, _dp, _dp, _i64p]
        L.rspr_decompose_uniform.restype = ct.c_int
        L.rspr_bench_matvec.argtypes = [ct.c_size_t, ct.c_size_t, ct.c_double, ct.c_size_t,
                                        ct.c_uint64, ct.POINTER(ct.c_double),
                                        ct.POINTER(ct.c_double), _u64p, _u64p]
        L.rspr_bench_matvec.restype = ct.c_int
        L.rspr_write_layer.argtypes = [ct.c_void_p, _i64p, ct.c_char_p]
        L.rspr_write_layer.restype = ct.c_int
        L.rspr_read_layer.argtypes = [ct.c_char_p, _u64p, _dp, _dp, _dp, _i64p, _dp]
        L.rspr_read_layer.restype = ct.c_int
        L.rspr_mlp_forward.argtypes = [ct.c_void_p, ct.c_void_p, ct.c_void_p, _dp, ct.c_size_t, _dp]
        L.rspr_mlp_forward.restype = ct.c_int
        _ip = ct.POINTER(ct.c_int)
        _vpp = ct.POINTER(ct.c_void_p)
        L.rspr_model_write.argtypes = [ct.c_size_t] * 5 + [ct.c_uint64, ct.c_size_t, ct.c_char_p]
        L.rspr_model_write.restype = ct.c_int
        L.rspr_model_logits.argtypes = [ct.c_char_p, _ip, ct.c_size_t, _vpp, ct.c_size_t, ct.c_size_t, _dp]
        L.rspr_model_logits.restype = ct.c_int
        L.rspr_model_perplexity.argtypes = [ct.c_char_p, _ip, ct.c_size_t, ct.c_size_t, _vpp, ct.c_size_t, _dp]
        L.rspr_model_perplexity.restype = ct.c_int
        L.rspr_recipe_loss.argtypes = [ct.c_char_p, _ip, ct.c_size_t, ct.c_size_t, _dp, _dp, ct.c_size_t, _dp, _dp]
        L.rspr_recipe_loss.restype = ct.c_int
        L.rspr_aggregate_scores.argtypes = [_dp, ct.c_size_t, ct.c_size_t, _dp, _dp, ct.c_size_t,
                                            ct.c_uint, _dp]
        L.rspr_aggregate_scores.restype = ct.c_int
        L.rspr_select_components.argtypes = [_dp, ct.c_size_t, ct.c_size_t, ct.c_size_t, _i64p]
        L.rspr_select_components.restype = ct.c_int
        L.rspr_decompose_with_svd.argtypes = [_dp, ct.c_size_t, ct.c_size_t, ct.c_double, ct.c_size_t,
                                              _dp, ct.c_size_t, _dp, _dp, _dp, _dp, _dp, _i64p]
        L.rspr_decompose_with_svd.restype = ct.c_int

    class Layer:
        """An owned reference DecomposedLayer."""

        def __init__(self, ref: "RefOracle", w_cols, a_r, b_r, keep_fraction: float):
            w_cols, a_r, b_r = _as_f64(w_cols), _as_f64(a_r), _as_f64(b_r)
            self.m_in, self.m_out = w_cols.shape
            self.rank = a_r.shape[1] if a_r.ndim == 2 else 0
            self._ref = ref
            self.h = ref.lib.rspr_layer_create(self.m_in, self.m_out, self.rank, keep_fraction,
                                               _d(w_cols), _d(a_r), _d(b_r))
            if not self.h:
                raise UsageError(2, "rspr_layer_create")

        def forward(self, x) -> np.ndarray:
            x = _as_f64(x)
            y = np.empty(max(self.m_out, 1), dtype=np.float64)
            if x.size != self.m_in:
                raise UsageError(2, "forward: input length mismatch")
            _raise(self._ref.lib.rspr_layer_forward(self.h, _d(x), _d(y)), "forward")
            return y[: self.m_out].copy()

        def __del__(self):
            if getattr(self, "h", None):
                self._ref.lib.rspr_layer_destroy(self.h)
                self.h = None

    def layer(self, w_cols, a_r, b_r, keep_fraction: float) -> "RefOracle.Layer":
        return RefOracle.Layer(self, w_cols, a_r, b_r, keep_fraction)

    def forward(self, w_cols, a_r, b_r, keep_fraction: float, x) -> np.ndarray:
        return self.layer(w_cols, a_r, b_r, keep_fraction).forward(x)

    def forward_many(self, layers, xs, ys, threads: int) -> None:
        """layers: list of RefOracle.Layer; xs/ys preallocated float64 arrays."""
        hp = (ct.c_void_p * len(layers))(*[l.h for l in layers])
        xp = (_dp * len(xs))(*[_d(x) for x in xs])
        yp = (_dp * len(ys))(*[_d(y) for y in ys])
        _raise(self.lib.rspr_forward_many(hp, xp, yp, len(layers), threads), "forward_many")

    def matvec(self, w, x):
        w, x = _as_f64(w), _as_f64(x)
        y = np.empty(w.shape[0], dtype=np.float64)
        _raise(self.lib.rspr_matvec(_d(w), w.shape[0], w.shape[1], _d(x), _d(y)), "matvec")
        return y

    def plan_for(self, rho: float, budget: float, m_in: int, m_out: int):
        s, r = ct.c_double(), ct.c_size_t()
        self.lib.rspr_plan_for(rho, budget, m_in, m_out, ct.byref(s), ct.byref(r))
        return s.value, r.value

    def decompose_uniform(self, w, keep_fraction: float, rank: int):
        """Reference Jacobi-SVD decomposition (uniform score): returns a_r, b_r, comps."""
        w = _as_f64(w)
        m, n = w.shape
        a = np.empty(max(m * rank, 1), dtype=np.float64)
        b = np.empty(max(rank * n, 1), dtype=np.float64)
        comps = np.empty(max(rank, 1), dtype=np.int64)
        _raise(self.lib.rspr_decompose_uniform(_d(w), m, n, keep_fraction, rank, _d(a), _d(b),
                                               comps.ctypes.data_as(_i64p)), "decompose")
        return (a[: m * rank].reshape(m, rank).copy(), b[: rank * n].reshape(rank, n).copy(),
                comps[:rank].copy())

    def mlp_forward(self, up: "RefOracle.Layer", gate: "RefOracle.Layer", down: "RefOracle.Layer", x) -> np.ndarray:
        """mlp_forward (model.cpp:115-127): down(up(x) * silu(gate(x)))."""
        x = _as_f64(x)
        out = np.empty(x.shape[0], dtype=np.float64)
        _raise(self.lib.rspr_mlp_forward(up.h, gate.h, down.h, _d(x), x.shape[0], _d(out)), "mlp_forward")
        return out

    # -- model.cpp / search.cpp (the toy decoder that calls forward) ---------
    def model_write(self, path: str, num_layers=2, embed=64, hidden=172, heads=4, vocab=256, seed=1,
                    max_seq=256) -> None:
        """init_model + write_model (model.cpp:89-113, 767-792)."""
        _raise(self.lib.rspr_model_write(num_layers, embed, hidden, heads, vocab, seed, max_seq, path.encode()),
               "model_write")

    @staticmethod
    def _handles(layers):
        if layers is None:
            return None, 0
        arr = (ct.c_void_p * len(layers))(*[l.h for l in layers])
        return arr, len(layers)

    def model_logits(self, path: str, tokens, layers=None, decode_start: int = 0, vocab: int = 256) -> np.ndarray:
        """read_model + model_forward (model.cpp:159-242)."""
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        out = np.empty((tok.size, vocab), dtype=np.float64)
        hp, nl = self._handles(layers)
        _raise(self.lib.rspr_model_logits(path.encode(), tok.ctypes.data_as(ct.POINTER(ct.c_int)), tok.size, hp, nl,
                                          decode_start, _d(out)), "model_forward")
        return out

    def model_perplexity(self, path: str, tokens, split_point: int, layers=None) -> float:
        """read_model + perplexity (model.cpp:244-269)."""
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        out = ct.c_double()
        hp, nl = self._handles(layers)
        _raise(self.lib.rspr_model_perplexity(path.encode(), tok.ctypes.data_as(ct.POINTER(ct.c_int)), tok.size,
                                              split_point, hp, nl, ct.byref(out)), "perplexity")
        return out.value

    def recipe_loss(self, path: str, calib, seq_len: int, rho, budget):
        """RecipeEvaluator(model, calib, seq_len).loss(Recipe{rho, budget}), dense_loss() (search.cpp:36-105)."""
        tok = np.ascontiguousarray(calib, dtype=np.int32)
        r, b = _as_f64(rho), _as_f64(budget)
        loss, dense = ct.c_double(), ct.c_double()
        _raise(self.lib.rspr_recipe_loss(path.encode(), tok.ctypes.data_as(ct.POINTER(ct.c_int)), tok.size, seq_len,
                                         _d(r), _d(b), r.size, ct.byref(loss), ct.byref(dense)), "recipe_loss")
        return loss.value, dense.value

    def aggregate_scores(self, tokens, sigma, vt, workers: int = 1) -> np.ndarray:
        """aggregate_scores (scores.cpp:52-62): tokens [T, n], sigma [kc], vt [kc, n] -> [kc, n]."""
        tokens, sigma, vt = _as_f64(tokens), _as_f64(sigma), _as_f64(vt)
        T, n = tokens.shape
        kc = sigma.shape[0]
        out = np.empty(kc * n, dtype=np.float64)
        _raise(self.lib.rspr_aggregate_scores(_d(tokens), T, n, _d(sigma), _d(vt), kc, workers, _d(out)),
               "aggregate_scores")
        return out.reshape(kc, n)

    def select_components(self, scores, r: int) -> np.ndarray:
        """select_components (scores.cpp:73-85) -> ascending component indices."""
        scores = _as_f64(scores)
        kc, n = scores.shape
        comps = np.empty(max(r, 1), dtype=np.int64)
        _raise(self.lib.rspr_select_components(_d(scores), kc, n, r, comps.ctypes.data_as(_i64p)),
               "select_components")
        return comps[:r].copy()

    def decompose_with_svd(self, w, keep_fraction: float, rank: int, scores, u, sigma, vt):
        """decompose_with_svd (layer.cpp:35-68) -> a_r, b_r, comps."""
        w, scores, u, sigma, vt = (_as_f64(a) for a in (w, scores, u, sigma, vt))
        m, n = w.shape
        kc = sigma.shape[0]
        a = np.empty(max(m * rank, 1), dtype=np.float64)
        b = np.empty(max(rank * n, 1), dtype=np.float64)
        comps = np.empty(max(rank, 1), dtype=np.int64)
        _raise(self.lib.rspr_decompose_with_svd(_d(w), m, n, keep_fraction, rank, _d(scores), kc, _d(u), _d(sigma),
                                                _d(vt), _d(a), _d(b), comps.ctypes.data_as(_i64p)),
               "decompose_with_svd")
        return (a[: m * rank].reshape(m, rank).copy(), b[: rank * n].reshape(rank, n).copy(), comps[:rank].copy())

    def write_layer(self, path: str, w_cols, a_r, b_r, keep_fraction: float, comps=None) -> None:
        """write_decomposed_layer (layer.cpp:243-267) of the layer built from these arrays."""
        L = self.layer(w_cols, a_r, b_r, keep_fraction)
        cp = None
        if comps is not None:
            comps = np.ascontiguousarray(np.asarray(comps, dtype=np.int64))
            cp = comps.ctypes.data_as(_i64p)
        _raise(self.lib.rspr_write_layer(L.h, cp, path.encode()), "write_decomposed_layer")

    def read_layer(self, path: str):
        """read_decomposed_layer (layer.cpp:269-301) -> dict of arrays (float64)."""
        dims = (ct.c_uint64 * 3)()
        _raise(self.lib.rspr_read_layer(path.encode(), dims, None, None, None, None, None),
               "read_decomposed_layer")
        n, m, r = int(dims[0]), int(dims[1]), int(dims[2])
        w = np.empty(max(n * m, 1)); a = np.empty(max(m * r, 1)); b = np.empty(max(r * n, 1))
        comps = np.empty(max(r, 1), dtype=np.int64)
        plan = np.empty(2)
        _raise(self.lib.rspr_read_layer(path.encode(), dims, _d(w), _d(a), _d(b),
                                        comps.ctypes.data_as(_i64p), _d(plan)), "read_decomposed_layer")
        return {"m_in": n, "m_out": m, "rank": r, "w_cols": w[: n * m].reshape(n, m).copy(),
                "a_r": a[: m * r].reshape(m, r).copy(), "b_r": b[: r * n].reshape(r, n).copy(),
                "comps": comps[:r].copy(), "keep_fraction": float(plan[0])}

    def bench_matvec(self, m_in: int, m_out: int, s: float, reps: int, seed: int = 42):
        dn, gn = ct.c_double(), ct.c_double()
        db, tb = ct.c_uint64(), ct.c_uint64()
        _raise(self.lib.rspr_bench_matvec(m_in, m_out, s, reps, seed, ct.byref(dn), ct.byref(gn),
                                          ct.byref(db), ct.byref(tb)), "bench_matvec")
        return {"dense_ns_median": dn.value, "gather_ns_median": gn.value,
                "dense_bytes": db.value, "touched_bytes": tb.value}


_C = None
_REF = None


def c_oracle() -> COracle:
    global _C
    if _C is None:
        if not os.path.exists(C_PATH):
            build()
        _C = COracle()
    return _C


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref_oracle() -> RefOracle:
    global _REF
    if _REF is None:
        _REF = RefOracle()
    return _REF
