"""Offline factor build on the GPU: the step before the path.

Mirrors the reference's decomposition API over the C ABI (fp64 device
buffers, kernels in csrc/rsp_offline.cu):

* ``SvdResult`` -- ``svd.hpp:12-21`` (u m x kc, sigma kc, vt kc x n);
* ``svd(w)`` -- the thin SVD of ``w`` by cuSOLVER (``torch.linalg.svd`` on
  the device), in place of the reference's one-sided Jacobi
  (``svd.cpp:21-173``, hours at 4096^2);
* ``score_single_token`` / ``aggregate_scores`` -- ``scores.cpp:15-62``
  (bit-identical to the reference for the same SVD);
* ``select_components`` -- ``scores.cpp:73-85``;
* ``decompose_with_svd`` / ``decompose`` -- ``layer.cpp:35-72``: returns a
  device-resident :class:`DecomposedLayer` whose ``selected_components``
  are the chosen components.

Errors follow the reference's exceptions (``UsageError`` for an empty token
list, r > component count, a score shape that does not match the weight).
"""
from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass
from typing import List, Sequence

import torch

from . import _lib as L
from ._lib import check
from .layer import DecomposedLayer, SparsityPlan, _stream_ptr


def _dev64(a, device) -> torch.Tensor:
    t = a if isinstance(a, torch.Tensor) else torch.as_tensor(a)
    return t.to(device=device, dtype=torch.float64).contiguous()


def _device(device) -> torch.device:
    if isinstance(device, torch.device):
        return device
    return torch.device("cuda", int(device)) if not isinstance(device, str) else torch.device(device)


@dataclass
class SvdResult:
    """svd.hpp:12-21: w = u diag(sigma) vt (fp64, on the device)."""
    u: torch.Tensor
    sigma: torch.Tensor
    vt: torch.Tensor

    def num_components(self) -> int:
        return int(self.sigma.shape[0])

    def reconstruct(self) -> torch.Tensor:
        return (self.u * self.sigma) @ self.vt


@dataclass
class ScoreMatrix:
    """scores.hpp:15-19."""
    values: torch.Tensor  # [num_components, m_in] fp64
    token_count: int
    layer_id: str = ""


def svd(w, device=0) -> SvdResult:
    """Thin SVD of an m x n weight (cuSOLVER through torch.linalg.svd, fp64)."""
    W = _dev64(w, _device(device))
    u, s, vt = torch.linalg.svd(W, full_matrices=False)
    return SvdResult(u.contiguous(), s.contiguous(), vt.contiguous())


def aggregate_scores(tokens: Sequence, svd_result: SvdResult, layer_id: str = "",
                     num_workers: int = 1, stream=None) -> ScoreMatrix:
    """scores.cpp:52-62: mean over tokens of |sigma_i x_j Vt_ij| (``num_workers``
    is accepted for API parity; the result never depends on it)."""
    if len(tokens) == 0:
        raise L.UsageError(L.RSP_E_USAGE, "aggregate_scores requires at least one token")
    dev = svd_result.vt.device
    X = torch.stack([_dev64(t, dev) for t in tokens]) if not isinstance(tokens, torch.Tensor) else _dev64(tokens, dev)
    T, n = int(X.shape[0]), int(X.shape[1])
    kc = svd_result.num_components()
    if n != int(svd_result.vt.shape[1]):
        raise L.UsageError(L.RSP_E_USAGE, f"score_single_token: input length {n} does not match V rows "
                                          f"{int(svd_result.vt.shape[1])}")
    sig, vt = _dev64(svd_result.sigma, dev), _dev64(svd_result.vt, dev)
    out = torch.empty((kc, n), dtype=torch.float64, device=dev)
    check(L.lib().rsp_aggregate_scores(X.data_ptr(), T, n, sig.data_ptr(), vt.data_ptr(), kc, out.data_ptr(),
                                       _stream_ptr(stream)), "aggregate_scores")
    return ScoreMatrix(out, T, layer_id)


def score_single_token(x, svd_result: SvdResult, stream=None) -> torch.Tensor:
    """scores.cpp:15-29 (signed): s[i][j] = sigma_i x_j Vt_ij."""
    dev = svd_result.vt.device
    x = _dev64(x, dev)
    if x.shape[0] != svd_result.vt.shape[1]:
        raise L.UsageError(L.RSP_E_USAGE, f"score_single_token: input length {int(x.shape[0])} does not match "
                                          f"V rows {int(svd_result.vt.shape[1])}")
    return (svd_result.sigma.to(dev, torch.float64)[:, None] * x[None, :]) * svd_result.vt.to(dev, torch.float64)


def select_components(scores: ScoreMatrix, r: int, stream=None) -> List[int]:
    """scores.cpp:73-85: the r components of largest row mass, ascending."""
    vals = scores.values if isinstance(scores, ScoreMatrix) else scores
    vals = vals.to(torch.float64).contiguous()
    kc, n = int(vals.shape[0]), int(vals.shape[1])
    dev = vals.device
    comps = torch.empty(max(r, 1), dtype=torch.int32, device=dev)
    mass = torch.empty(max(kc, 1), dtype=torch.float64, device=dev)
    check(L.lib().rsp_select_components(vals.data_ptr(), kc, n, r, comps.data_ptr(), mass.data_ptr(),
                                        _stream_ptr(stream)), "select_components")
    return comps[:r].cpu().tolist()


def _split(svd_result: SvdResult, comps: List[int], m: int, n: int, stream=None):
    dev = svd_result.vt.device
    r = len(comps)
    u, sig, vt = (_dev64(a, dev) for a in (svd_result.u, svd_result.sigma, svd_result.vt))
    a_r = torch.empty((m, r), dtype=torch.float64, device=dev)
    b_r = torch.empty((r, n), dtype=torch.float64, device=dev)
    cd = torch.tensor(comps if r else [0], dtype=torch.int32, device=dev)
    check(L.lib().rsp_split_factors(u.data_ptr(), m, int(u.shape[1]), sig.data_ptr(), vt.data_ptr(), n,
                                    cd.data_ptr(), r, a_r.data_ptr(), b_r.data_ptr(), _stream_ptr(stream)),
          "split_factors")
    return a_r, b_r


def decompose_with_svd(w, plan: SparsityPlan, scores: ScoreMatrix, svd_result: SvdResult, *,
                       stream=None, **layer_kw) -> DecomposedLayer:
    """layer.cpp:35-68 -> a device-resident DecomposedLayer (``layer_kw`` as
    :class:`DecomposedLayer`: weight_dtype, k, device, shard_rank, ...)."""
    m_out, m_in = int(w.shape[0]), int(w.shape[1])
    kc = min(m_in, m_out)
    r = int(plan.rank)
    if r > kc:
        raise L.UsageError(L.RSP_E_USAGE, f"decompose: rank {r} exceeds min(m_in, m_out) = {kc}")
    vals = scores.values if isinstance(scores, ScoreMatrix) else scores
    if tuple(vals.shape) != (kc, m_in):
        raise L.UsageError(L.RSP_E_USAGE, f"decompose: score shape {int(vals.shape[0])}x{int(vals.shape[1])} does "
                                          f"not match SVD of a {m_out}x{m_in} weight")
    comps = select_components(scores, r, stream=stream)
    a_r, b_r = _split(svd_result, comps, m_out, m_in, stream=stream)
    torch.cuda.synchronize(svd_result.vt.device)
    W = _dev64(w, svd_result.vt.device)
    layer = DecomposedLayer(W, a_r if r else None, b_r if r else None, plan, **layer_kw)
    if r:
        buf = (ct.c_uint32 * r)(*comps)
        check(L.lib().rsp_linear_set_components(layer.handle, buf, r), "set_components")
    return layer


def decompose(w, plan: SparsityPlan, scores: ScoreMatrix, *, device=0, stream=None,
              **layer_kw) -> DecomposedLayer:
    """layer.cpp:70-72: SVD of ``w`` (cuSOLVER) then :func:`decompose_with_svd`."""
    s = svd(w, device=device)
    dev = _device(device)
    return decompose_with_svd(w, plan, scores, s, stream=stream, device=dev.index or 0, **layer_kw)


def uniform_scores(m_out: int, m_in: int, device=0) -> ScoreMatrix:
    """A uniform score (test_layer.cpp:19-22): selects the leading components."""
    kc = min(m_out, m_in)
    return ScoreMatrix(torch.ones((kc, m_in), dtype=torch.float64, device=_device(device)), 1, "")
