"""Seeded synthetic inputs for the BASELINE.json configurations.

No public dataset is involved in this path: these
generators ARE the workload.  Decisions recorded in DESIGN.md:

* W = 0.02 N(0,1) + L R with L (m x 256), R (256 x n) entries N(0, 0.01)
  read as variance 0.01 (std 0.1) -- the reading that gives the "decaying
  spectrum" the config asks for.
* "scaled per matrix" (configs 1/2): each matrix is multiplied by a seeded
  constant drawn from U(0.5, 1.5).
* x_j = Laplace(0,1) * LogNormal(0,1), plus `outliers` distinct random
  channels scaled x20 (config 0; 16 outliers in config 4).
* down_proj input = SiLU(g) * u with g, u ~ N(0,1) (config 1).
* Config 2 per-layer plans: rho ~ U(0.3, 0.7), budget C = 0.5 through
  Recipe::plan_for (search.cpp:14-25): s = 0.5 rho, r = round((1-rho) C mn/(m+n)).
"""
from __future__ import annotations

from typing import Dict, List, Tuple

import zlib

import numpy as np

# Llama-2-7B decoder-layer linears: (name, m_out, m_in)
LLAMA2_7B = [
    ("q_proj", 4096, 4096), ("k_proj", 4096, 4096), ("v_proj", 4096, 4096),
    ("o_proj", 4096, 4096), ("gate_proj", 11008, 4096), ("up_proj", 11008, 4096),
    ("down_proj", 4096, 11008),
]
# Llama-3-8B (GQA): k/v are 1024 x 4096
LLAMA3_8B = [
    ("q_proj", 4096, 4096), ("k_proj", 1024, 4096), ("v_proj", 1024, 4096),
    ("o_proj", 4096, 4096), ("gate_proj", 14336, 4096), ("up_proj", 14336, 4096),
    ("down_proj", 4096, 14336),
]
N_LAYERS = 32

# Which input each decoder-layer linear reads (model.cpp:159-242 decode
# order): q/k/v share the normed hidden state, o reads the attention
# context, gate/up share the post-attention normed state, down reads
# up * SiLU(gate).  A linear that starts a new input group depends on the
# previous linear's output in a real decode (wait_prev); the others may
# overlap with the linear before them.
INPUT_GROUP = {"q_proj": "attn_in", "k_proj": "attn_in", "v_proj": "attn_in", "o_proj": "attn_out",
               "gate_proj": "mlp_in", "up_proj": "mlp_in", "down_proj": "mlp_act"}


def input_groups(plans):
    """[(group index per linear)], [wait_prev per linear]: consecutive linears
    of one decoder layer reading the same input share one activation vector."""
    gid, wait, last = [], [], None
    for (name, *_rest) in plans:
        layer, short = name.rsplit(".", 1) if "." in name else ("", name)
        key = (layer, INPUT_GROUP.get(short, short))
        if key != last:
            gid.append(gid[-1] + 1 if gid else 0)
            wait.append(True)
            last = key
        else:
            gid.append(gid[-1])
            wait.append(False)
    return gid, wait


def heavy_tailed_x(n: int, rng: np.random.Generator, outliers: int = 8, scale: float = 20.0) -> np.ndarray:
    """Laplace(0,1) * LogNormal(0,1) with `outliers` channels x`scale` (float32)."""
    x = rng.laplace(0.0, 1.0, n) * rng.lognormal(0.0, 1.0, n)
    if outliers:
        idx = rng.choice(n, size=min(outliers, n), replace=False)
        x[idx] *= scale
    return x.astype(np.float32)


def silu_gate_x(n: int, rng: np.random.Generator) -> np.ndarray:
    """down_proj input SiLU(g) * u, g, u ~ N(0,1) (model.cpp:122-126 semantics)."""
    g = rng.standard_normal(n)
    u = rng.standard_normal(n)
    return (g / (1.0 + np.exp(-g)) * u).astype(np.float32)


def structured_weight(m: int, n: int, rng: np.random.Generator, inner: int = 256,
                      scale: float = 1.0) -> np.ndarray:
    """W = scale * (0.02 N(0,1) + L R), L: m x inner, R: inner x n, entries std 0.1 (float32)."""
    Lm = (rng.standard_normal((m, inner)) * 0.1).astype(np.float32)
    Rm = (rng.standard_normal((inner, n)) * 0.1).astype(np.float32)
    w = (rng.standard_normal((m, n)) * 0.02).astype(np.float32)
    w += Lm @ Rm
    if scale != 1.0:
        w *= np.float32(scale)
    return w


def svd_factors(w, r: int):
    """a_r = U_r sqrt(S_r) (m x r), b_r = sqrt(S_r) Vt_r (r x n) -- the
    reference's split (layer.cpp:61-66) of a truncated SVD (uniform score).
    Accepts numpy or torch (runs on the tensor's device)."""
    import torch
    t = torch.as_tensor(w)
    if r == 0:
        m, n = t.shape
        return t.new_zeros((m, 0)), t.new_zeros((0, n))
    U, S, Vh = torch.linalg.svd(t.double() if not t.is_cuda else t.float(), full_matrices=False)
    root = S[:r].sqrt()
    a = U[:, :r] * root[None, :]
    b = root[:, None] * Vh[:r, :]
    return a.to(t.dtype), b.to(t.dtype)


def config0(seed: int = 0, m: int = 4096, n: int = 4096, r: int = 256, k: int = 2048,
            outliers: int = 8, device: str = "cpu") -> Dict:
    """Config 0: single fp32 linear, truncated-SVD factors, heavy-tailed x."""
    import torch
    rng = np.random.default_rng(seed)
    w = structured_weight(m, n, rng)
    x = heavy_tailed_x(n, rng, outliers)
    wt = torch.from_numpy(w).to(device)
    a, b = svd_factors(wt, r)
    return {"w": wt, "a_r": a, "b_r": b, "x": torch.from_numpy(x).to(device), "k": k,
            "keep_fraction": k / n, "rank": r}


def config1_layer(name: str, m: int, n: int, seed: int = 1, device: str = "cpu") -> Dict:
    """Config 1: one Llama-2-7B linear, s = 0.5, r = n/16, scaled per matrix."""
    import torch
    rng = np.random.default_rng([seed, m, n, zlib.crc32(name.encode())])
    scale = float(rng.uniform(0.5, 1.5))
    w = structured_weight(m, n, rng, scale=scale)
    x = silu_gate_x(n, rng) if name == "down_proj" else heavy_tailed_x(n, rng)
    r = n // 16
    wt = torch.from_numpy(w).to(device)
    a, b = svd_factors(wt, r)
    return {"name": name, "w": wt, "a_r": a, "b_r": b, "x": torch.from_numpy(x).to(device),
            "keep_fraction": 0.5, "rank": r, "scale": scale}


def config2_plans(seed: int = 2, budget: float = 0.5, shapes=LLAMA2_7B,
                  n_layers: int = N_LAYERS) -> List[Tuple[str, int, int, float, int]]:
    """Per-linear (name, m_out, m_in, keep_fraction, rank) for the config-2
    stack: rho ~ U(0.3, 0.7) per linear, C = budget, Recipe::plan_for."""
    from .layer import Recipe
    rng = np.random.default_rng(seed)
    out = []
    for layer in range(n_layers):
        for (name, m, n) in shapes:
            rho = float(rng.uniform(0.3, 0.7))
            plan = Recipe([rho], [budget]).plan_for(0, n, m)
            out.append((f"layers.{layer}.{name}", m, n, plan.keep_fraction, plan.rank))
    return out


def config4_plans(sparsity: float, rank: int, n_layers: int = N_LAYERS):
    """Config 4 (BASELINE.json configs[4]): the Llama-3-8B stack at model-level
    sparsity `sparsity` with every linear at rank `rank`: keep fraction
    s = (1 - sparsity) - r (m + n) / (m n) so each linear's reference io_cost
    is 1 - sparsity.  Where that s is negative (GQA k/v at
    high sparsity / rank) the rank is clamped to floor((1 - sparsity) m n /
    (m + n)) with s = 0, and the clamp is reported: returns (plans, clamped)."""
    out, clamped = [], []
    for layer in range(n_layers):
        for (name, m, n) in LLAMA3_8B:
            r = rank
            s = (1.0 - sparsity) - r * (m + n) / (m * n)
            if s < 0.0:
                r = int(np.floor((1.0 - sparsity) * m * n / (m + n)))
                s = 0.0
                if layer == 0:
                    clamped.append((name, rank, r))
            out.append((f"layers.{layer}.{name}", m, n, float(s), int(r)))
    return out, clamped


def stack_bytes(plans, elem: int = 2) -> Tuple[int, int]:
    """(R-Sparse kernel weight bytes, dense bytes) for a list of plans, using
    the SURVEY §8(d) byte model elem*(k*m + (n-k)*r + r*m) vs elem*m*n."""
    sparse = dense = 0
    for (_, m, n, s, r) in plans:
        k = int(np.ceil(s * n))
        sparse += elem * (k * m + ((n - k) * r + r * m if (r > 0 and k < n) else 0))
        dense += elem * m * n
    return sparse, dense
