"""Model-level callers of the operator (model.cpp:115-141).

The reference's decoder calls ``forward`` once per linear (``apply_linear``)
and builds the MLP input of ``down_proj`` as ``up(x) * silu(gate(x))``
(``mlp_forward``).  These mirrors run the same dataflow on the device: each
linear through the R-Sparse kernels (or, for dense positions, the dense
kernel), the gating elementwise in between.
"""
from __future__ import annotations

import torch

from . import _lib as L
from .layer import DecomposedLayer


def silu(z: torch.Tensor) -> torch.Tensor:
    """model.cpp:70: z / (1 + exp(-z))."""
    return z / (1.0 + torch.exp(-z))


def apply_linear(layer: DecomposedLayer, u: torch.Tensor, decoded: bool = True, stream=None) -> torch.Tensor:
    """model.cpp:133-141: the decomposed forward in the decode region, else the
    dense product of the same (device-resident) weight."""
    return layer.forward(u, stream=stream) if decoded else layer.dense_forward(u, stream=stream)


def mlp_forward(x: torch.Tensor, up: DecomposedLayer, gate: DecomposedLayer, down: DecomposedLayer,
                stream=None) -> torch.Tensor:
    """model.cpp:115-127: down(up(x) * silu(gate(x))) with x of length up.m_in."""
    if x.shape[-1] != up.m_in:
        raise L.UsageError(L.RSP_E_USAGE, f"mlp_forward: input length {int(x.shape[-1])} does not match "
                                          f"embed dim {up.m_in}")
    up_h = up.forward(x, stream=stream)
    gate_h = gate.forward(x, stream=stream)
    return down.forward(up_h * silu(gate_h), stream=stream)
