"""Model-level callers of the operator: the reference's toy
decoder (``rsparse::ToyModel``, model.hpp:45-57) resident on the device, with
every linear of the decode region run through the R-Sparse kernels.

* :func:`apply_linear` / :func:`mlp_forward` -- model.cpp:115-141.
* :class:`ToyModel` -- the weights of a reference model, loaded from its RSPW
  file (``write_model`` / ``read_model``, model.cpp:735-849).
* :class:`DecodeBlock` -- one block's seven decomposed linears as two
  persistent stack launches per decode position: q/k/v side by side (one
  shared input), and the whole gated MLP -- gate and up side by side, then
  down, whose input ``up * silu(gate)`` is formed inside the kernel's x load
  (``RSP_XOP_SILU_GATE``) from the outputs the same launch just produced: the
  y -> x dataflow of model.cpp:115-127 without leaving the kernel.  o_proj
  (after the attention) is a single forward.
* :func:`model_forward`, :func:`perplexity` -- model.cpp:159-269: positions
  before ``decode_start`` run dense (the prefill), the rest through the
  decomposed layers; attention, norms, embeddings and the head are fp64 on
  the device, as the reference computes them in double.
* :class:`RecipeEvaluator` -- search.cpp:36-105: calibration inputs from the
  dense model, one SVD (cuSOLVER) and one score matrix per linear, ``build``
  = decompose_with_svd per linear at ``Recipe.plan_for``, ``loss`` = mean
  perplexity with the prefill/decode split at half of each sequence.
"""
from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib as L
from .layer import DecomposedLayer, Recipe, Stack

KRMS_EPS = 1e-6  # model.cpp:66
SLOTS = ("q", "k", "v", "o", "up", "gate", "down")  # LinearSlot order (model.hpp:30)


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


# --------------------------------------------------------------------------- the toy model
@dataclass
class ModelConfig:
    """model.hpp:14-23."""
    num_layers: int = 4
    embed_dim: int = 64
    hidden_dim: int = 172
    num_heads: int = 4
    vocab_size: int = 256
    seed: int = 1
    max_seq: int = 256

    def validate(self) -> None:  # model.cpp:13-23
        if self.num_layers == 0:
            raise L.UsageError(L.RSP_E_USAGE, "model needs at least one block")
        if self.num_heads == 0 or self.embed_dim % self.num_heads:
            raise L.UsageError(L.RSP_E_USAGE, "embed_dim must be divisible by num_heads")
        if self.hidden_dim <= self.embed_dim:
            raise L.UsageError(L.RSP_E_USAGE, "hidden_dim must exceed embed_dim (gated MLP expansion)")
        if self.vocab_size < 2:
            raise L.UsageError(L.RSP_E_USAGE, "vocab_size must be at least 2")
        if self.max_seq == 0:
            raise L.UsageError(L.RSP_E_USAGE, "max_seq must be positive")


@dataclass
class ToyModel:
    """rsparse::ToyModel on the device (fp64 tensors: the values the RSPW file
    stores, widened exactly like read_model does)."""
    config: ModelConfig
    token_embedding: torch.Tensor     # vocab x n
    position_embedding: torch.Tensor  # max_seq x n
    blocks: List[dict]                # per block: q,k,v,o,up,gate,down (m x n), ln1, ln2
    final_gain: torch.Tensor          # n
    head: torch.Tensor                # vocab x n
    device: torch.device = field(default_factory=lambda: torch.device("cuda", 0))

    def num_linear_layers(self) -> int:
        return len(self.blocks) * len(SLOTS)

    def linear_weight(self, idx: int) -> torch.Tensor:
        """ToyModel::linear_weight (model.cpp:38-51): global index = block * 7 + slot."""
        return self.blocks[idx // 7][SLOTS[idx % 7]]

    def linear_name(self, idx: int) -> str:
        names = ("wq", "wk", "wv", "wo", "wup", "wgate", "wdown")
        return f"b{idx // 7}.{names[idx % 7]}"

    @classmethod
    def read_rspw(cls, path: str, device=0) -> "ToyModel":
        """read_model (model.cpp:794-849): magic RSPW, u8 version 1, u32 layers,
        embed, hidden, heads, vocab, u64 seed, u32 max_seq, then every tensor
        as little-endian f32 in declaration order."""
        if isinstance(device, torch.device):
            dev = device
        elif isinstance(device, str):
            dev = torch.device(device)
        else:
            dev = torch.device("cuda", int(device))
        with open(path, "rb") as f:
            buf = f.read()
        if len(buf) < 4 or buf[:4] != b"RSPW":
            raise L.IoError(L.RSP_E_IO, f"bad magic in {path} (expected RSPW)")
        if len(buf) < 5:
            raise L.IoError(L.RSP_E_IO, f"truncated file: {path}")
        if buf[4] != 1:
            raise L.IoError(L.RSP_E_IO, f"unsupported RSPW version {buf[4]} in {path}")
        hdr = struct.Struct("<IIIIIQI")
        if len(buf) < 5 + hdr.size:
            raise L.IoError(L.RSP_E_IO, f"truncated file: {path}")
        cfg = ModelConfig(*hdr.unpack_from(buf, 5))
        cfg.validate()
        off = 5 + hdr.size
        n, h = cfg.embed_dim, cfg.hidden_dim

        def take(*shape):
            nonlocal off
            cnt = int(np.prod(shape))
            if len(buf) < off + 4 * cnt:
                raise L.IoError(L.RSP_E_IO, f"truncated file: {path}")
            a = np.frombuffer(buf, dtype="<f4", count=cnt, offset=off).astype(np.float64).reshape(shape)
            off += 4 * cnt
            return torch.from_numpy(a).to(dev)

        tok = take(cfg.vocab_size, n)
        pos = take(cfg.max_seq, n)
        blocks = []
        for _ in range(cfg.num_layers):
            b = {"q": take(n, n), "k": take(n, n), "v": take(n, n), "o": take(n, n),
                 "up": take(h, n), "gate": take(h, n), "down": take(n, h)}
            b["ln1"] = take(n)
            b["ln2"] = take(n)
            blocks.append(b)
        fin = take(n)
        head = take(cfg.vocab_size, n)
        return cls(cfg, tok, pos, blocks, fin, head, dev)


def rms_normalize(x: torch.Tensor, gain: torch.Tensor) -> torch.Tensor:
    """model.cpp:78-86 (fp64): g * x / sqrt(mean(x^2) + 1e-6)."""
    rms = torch.sqrt((x * x).sum(-1, keepdim=True) / x.shape[-1] + KRMS_EPS)
    return gain * x / rms


class DecodeBlock:
    """One block's decomposed linears on persistent device buffers: the q/k/v
    stack, o_proj, and the MLP stack (gate | up side by side, then down with
    the SiLU gating fused into its x load)."""

    def __init__(self, layers: Sequence[DecomposedLayer], dev: torch.device):
        q, k, v, o, up, gate, down = layers
        n, h = q.m_in, up.m_out
        self.o = o
        self.u = torch.zeros(n, dtype=torch.float32, device=dev)      # normed hidden (q/k/v, gate/up input)
        self.yqkv = torch.zeros(3 * n, dtype=torch.float32, device=dev)
        self.yug = torch.zeros(2 * h, dtype=torch.float32, device=dev)  # [up | gate]: down's gated input
        self.ydown = torch.zeros(n, dtype=torch.float32, device=dev)
        self.qkv = Stack([q, k, v], [self.u] * 3, [self.yqkv[:n], self.yqkv[n:2 * n], self.yqkv[2 * n:]],
                         wait_prev=[True, False, False])
        # the x of down is self.yug: [a = up | g = gate], input a * silu(g) (RSP_XOP_SILU_GATE)
        self.mlp = Stack([gate, up, down], [self.u, self.u, self.yug], [self.yug[h:], self.yug[:h], self.ydown],
                         wait_prev=[True, False, True], silu_gate=[False, False, True])
        self.n = n

    def qkv_forward(self, u64: torch.Tensor):
        self.u.copy_(u64)
        self.qkv.launch()
        n = self.n
        return self.yqkv[:n].double(), self.yqkv[n:2 * n].double(), self.yqkv[2 * n:].double()

    def o_forward(self, ctx64: torch.Tensor) -> torch.Tensor:
        return self.o.forward(ctx64.float().contiguous()).double()

    def mlp_forward(self, u64: torch.Tensor) -> torch.Tensor:
        self.u.copy_(u64)
        self.mlp.launch()
        return self.ydown.double()

    def close(self):
        self.qkv.close()
        self.mlp.close()


def _check_tokens(model: ToyModel, tokens) -> None:  # model.cpp:143-155
    if len(tokens) == 0:
        raise L.UsageError(L.RSP_E_USAGE, "token sequence is empty")
    if len(tokens) > model.config.max_seq:
        raise L.UsageError(L.RSP_E_USAGE, f"sequence length {len(tokens)} exceeds max_seq {model.config.max_seq}")
    for t in tokens:
        if t < 0 or t >= model.config.vocab_size:
            raise L.UsageError(L.RSP_E_USAGE, f"token id {t} outside vocabulary of {model.config.vocab_size}")


def decode_blocks(model: ToyModel, layers: Sequence[DecomposedLayer]) -> List[DecodeBlock]:
    """The DecodeBlocks of a decomposed model (layers in global linear order)."""
    if len(layers) != model.num_linear_layers():
        raise L.UsageError(L.RSP_E_USAGE, f"decomposed model has {len(layers)} layers, model needs "
                                          f"{model.num_linear_layers()}")
    return [DecodeBlock(layers[7 * b: 7 * b + 7], model.device) for b in range(len(model.blocks))]


def model_forward(model: ToyModel, tokens: Sequence[int], layers: Optional[Sequence[DecomposedLayer]] = None,
                  decode_start: int = 0, blocks: Optional[List[DecodeBlock]] = None) -> torch.Tensor:
    """model.cpp:159-242: logits (T x vocab, fp64 on the device).  Positions
    >= decode_start run every linear through its decomposed form on the
    R-Sparse kernels; earlier positions (and all, without ``layers``) run the
    dense fp64 products (the prefill)."""
    _check_tokens(model, tokens)
    own = False
    if layers is not None and blocks is None:
        blocks, own = decode_blocks(model, layers), True
    T, n = len(tokens), model.config.embed_dim
    heads = model.config.num_heads
    hd = n // heads
    scale = 1.0 / math.sqrt(hd)
    dev = model.device
    tok = torch.as_tensor(list(tokens), device=dev, dtype=torch.long)
    x = model.token_embedding[tok] + model.position_embedding[:T]
    dec = [blocks is not None and p >= decode_start for p in range(T)]
    try:
        for bi, b in enumerate(model.blocks):
            db = blocks[bi] if blocks is not None else None
            u = rms_normalize(x, b["ln1"])
            q, k, v = u @ b["q"].T, u @ b["k"].T, u @ b["v"].T
            for p in range(T):
                if dec[p]:
                    q[p], k[p], v[p] = db.qkv_forward(u[p])
            # causal attention over all positions, fp64 (model.cpp:193-214)
            qh, kh, vh = (t.view(T, heads, hd).transpose(0, 1) for t in (q, k, v))
            w = (qh @ kh.transpose(1, 2)) * scale
            w = w.masked_fill(torch.triu(torch.ones(T, T, dtype=torch.bool, device=dev), 1), float("-inf"))
            w = torch.softmax(w, dim=-1)
            ctx = (w @ vh).transpose(0, 1).reshape(T, n)
            att = ctx @ b["o"].T
            for p in range(T):
                if dec[p]:
                    att[p] = db.o_forward(ctx[p])
            x = x + att
            u = rms_normalize(x, b["ln2"])
            mlp = (u @ b["up"].T * silu(u @ b["gate"].T)) @ b["down"].T
            for p in range(T):
                if dec[p]:
                    mlp[p] = db.mlp_forward(u[p])
            x = x + mlp
        u = rms_normalize(x, model.final_gain)
        return u @ model.head.T
    finally:
        if own:
            for db in blocks:
                db.close()


def perplexity(model: ToyModel, tokens: Sequence[int], split_point: int,
               layers: Optional[Sequence[DecomposedLayer]] = None,
               blocks: Optional[List[DecodeBlock]] = None) -> float:
    """model.cpp:244-269: exp(mean next-token NLL) over targets after
    split_point; positions before it run dense (prefill)."""
    if split_point >= len(tokens):
        raise L.UsageError(L.RSP_E_USAGE, f"split_point {split_point} must lie before the sequence end {len(tokens)}")
    first = split_point + 1
    if first >= len(tokens):
        raise L.UsageError(L.RSP_E_USAGE, f"no scored positions beyond split_point {split_point}")
    logits = model_forward(model, tokens, layers, split_point, blocks)
    rows = logits[first - 1: len(tokens) - 1]
    tgt = torch.as_tensor(list(tokens[first:]), device=logits.device, dtype=torch.long)
    logp = rows.gather(1, tgt[:, None])[:, 0] - torch.logsumexp(rows, dim=1)
    return float(torch.exp(-logp.mean()))


def collect_linear_inputs(model: ToyModel, tokens: Sequence[int]) -> List[torch.Tensor]:
    """model.cpp:271-347: the dense model's input to every linear at every
    position, out[linear] = (T x m_in) fp64."""
    _check_tokens(model, tokens)
    T, n = len(tokens), model.config.embed_dim
    heads = model.config.num_heads
    hd = n // heads
    dev = model.device
    tok = torch.as_tensor(list(tokens), device=dev, dtype=torch.long)
    x = model.token_embedding[tok] + model.position_embedding[:T]
    out: List[torch.Tensor] = []
    for b in model.blocks:
        u = rms_normalize(x, b["ln1"])
        q, k, v = u @ b["q"].T, u @ b["k"].T, u @ b["v"].T
        qh, kh, vh = (t.view(T, heads, hd).transpose(0, 1) for t in (q, k, v))
        w = (qh @ kh.transpose(1, 2)) / math.sqrt(hd)
        w = w.masked_fill(torch.triu(torch.ones(T, T, dtype=torch.bool, device=dev), 1), float("-inf"))
        ctx = (torch.softmax(w, dim=-1) @ vh).transpose(0, 1).reshape(T, n)
        x = x + ctx @ b["o"].T
        u2 = rms_normalize(x, b["ln2"])
        up, gate = u2 @ b["up"].T, u2 @ b["gate"].T
        hidden = up * silu(gate)
        x = x + hidden @ b["down"].T
        out += [u, u, u, ctx, u2, u2, hidden]  # q, k, v, o, up, gate, down
    return out


class RecipeEvaluator:
    """search.cpp:36-105 on the device: per linear one SVD (cuSOLVER, replacing
    the Jacobi svd) and one score matrix from the dense model's inputs over
    the calibration sequences; candidates cost decompose_with_svd + forward
    passes through the R-Sparse kernels."""

    def __init__(self, model: ToyModel, calibration_tokens: Sequence[int], sequence_length: int,
                 weight_dtype: str = "f32"):
        from . import offline
        if sequence_length < 2:
            raise L.UsageError(L.RSP_E_USAGE, "calibration sequences need length >= 2")
        num_seq = len(calibration_tokens) // sequence_length
        if num_seq == 0:
            raise L.UsageError(L.RSP_E_USAGE, "empty calibration set")
        self.model = model
        self.weight_dtype = weight_dtype
        self.sequences = [list(calibration_tokens[s * sequence_length:(s + 1) * sequence_length])
                          for s in range(num_seq)]
        inputs: List[List[torch.Tensor]] = [[] for _ in range(model.num_linear_layers())]
        for seq in self.sequences:
            for l, t in enumerate(collect_linear_inputs(model, seq)):
                inputs[l].append(t)
        self.svds, self.scores = [], []
        for l in range(model.num_linear_layers()):
            s = offline.svd(model.linear_weight(l), device=model.device)
            self.svds.append(s)
            self.scores.append(offline.aggregate_scores(torch.cat(inputs[l]), s, model.linear_name(l)))

    def num_layers(self) -> int:
        return len(self.svds)

    def build(self, recipe: Recipe) -> List[DecomposedLayer]:
        """search.cpp:74-88."""
        from . import offline
        if recipe.num_layers() != self.num_layers():
            raise L.UsageError(L.RSP_E_USAGE, f"recipe has {recipe.num_layers()} layers, model has "
                                              f"{self.num_layers()}")
        out = []
        for l in range(self.num_layers()):
            w = self.model.linear_weight(l)
            plan = recipe.plan_for(l, int(w.shape[1]), int(w.shape[0]))
            out.append(offline.decompose_with_svd(w, plan, self.scores[l], self.svds[l],
                                                  weight_dtype=self.weight_dtype,
                                                  device=self.model.device.index or 0))
        return out

    def loss(self, recipe: Recipe) -> float:
        """search.cpp:90-97: mean perplexity, prefill/decode split at half."""
        layers = self.build(recipe)
        blocks = decode_blocks(self.model, layers)
        try:
            acc = sum(perplexity(self.model, seq, len(seq) // 2, blocks=blocks) for seq in self.sequences)
        finally:
            for db in blocks:
                db.close()
        return acc / len(self.sequences)

    def dense_loss(self) -> float:
        """search.cpp:99-105."""
        return sum(perplexity(self.model, seq, len(seq) // 2) for seq in self.sequences) / len(self.sequences)
