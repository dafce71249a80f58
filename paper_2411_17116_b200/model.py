"""The reference's seeded byte-level decoder (ss/toy_model.py), on the GPU.

This is plumbing around the hot path: embeddings, RMSNorm, projections and the
SiLU FFN run as torch ops (cuBLAS); RoPE and every attention call go through
libstar_attn.so.  Weights are drawn by the device splitmix64 kernel in the
reference's declaration order, so they are bit-identical to init_model's.
The model computes in fp32; attention inputs are cast to the build precision
(numerics.default_dtype) before reaching the kernels.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch

from . import ops
from .errors import ConfigError, DomainError
from .numerics import Prng, RopeConfig, default_dtype, prng_fill

_M64 = (1 << 64) - 1
_RMS_EPS = 1e-6
_GAIN_JITTER = 0.1


@dataclass(frozen=True)
class ModelConfig:
    """ss/toy_model.py:37-63."""

    d_model: int
    heads: int
    layers: int
    vocab: int = 256
    ff_mult: int = 2
    seed: int = 0
    rope_theta: float = 10000.0

    def __post_init__(self):
        for name in ("d_model", "heads", "layers", "vocab", "ff_mult"):
            if getattr(self, name) < 1:
                raise ConfigError(f"model {name} must be >= 1")
        if self.d_model % self.heads != 0:
            raise ConfigError(f"heads ({self.heads}) must divide d_model ({self.d_model})")
        object.__setattr__(self, "seed", int(self.seed) & _M64)

    @property
    def head_dim(self) -> int:
        return self.d_model // self.heads

    @property
    def rope(self) -> RopeConfig:
        return RopeConfig(self.head_dim, self.rope_theta)


@dataclass(frozen=True, eq=False)
class LayerWeights:
    wq: torch.Tensor
    wk: torch.Tensor
    wv: torch.Tensor
    wo: torch.Tensor
    w1: torch.Tensor
    w2: torch.Tensor
    attn_gain: torch.Tensor
    ffn_gain: torch.Tensor


@dataclass(frozen=True, eq=False)
class ModelWeights:
    config: ModelConfig
    embedding: torch.Tensor
    layers: tuple
    final_gain: torch.Tensor


def init_model(cfg: ModelConfig, device="cuda") -> ModelWeights:
    """Deterministic weights from cfg.seed in declaration order (ss/toy_model.py:93-113)."""
    prng = Prng(cfg.seed)
    d, ff = cfg.d_model, cfg.ff_mult * cfg.d_model
    s = 1.0 / float(torch.tensor(d, dtype=torch.float64).sqrt())

    def fill(r, c, scale):
        return prng_fill(prng, r, c, scale, torch.float32, device)

    def gain():
        return (1.0 + fill(1, d, _GAIN_JITTER)).reshape(-1)

    emb = fill(cfg.vocab, d, s)
    layers = []
    for _ in range(cfg.layers):
        wq, wk, wv, wo = fill(d, d, s), fill(d, d, s), fill(d, d, s), fill(d, d, s)
        w1, w2 = fill(d, ff, s), fill(ff, d, s)
        layers.append(LayerWeights(wq, wk, wv, wo, w1, w2, gain(), gain()))
    return ModelWeights(cfg, emb, tuple(layers), gain())


def _rms_norm(x: torch.Tensor, gain: torch.Tensor) -> torch.Tensor:
    ms = (x * x).mean(dim=-1, keepdim=True)
    return x / torch.sqrt(ms + _RMS_EPS) * gain


def _silu(x: torch.Tensor) -> torch.Tensor:
    return x / (1.0 + torch.exp(-x))


AttendFn = Callable[[int, torch.Tensor, torch.Tensor, torch.Tensor], torch.Tensor]
# batched form used by the B200 path: (q [rows, H, hd], k, v) -> out [rows, H, hd]
AttendAllFn = Callable[[torch.Tensor, torch.Tensor, torch.Tensor], torch.Tensor]


def embed(weights: ModelWeights, tokens) -> torch.Tensor:
    """Embedding rows for a token sequence (ss/toy_model.py:128-138)."""
    ids = [int(t) for t in tokens]
    if not ids:
        raise DomainError("cannot embed an empty token sequence")
    for t in ids:
        if not 0 <= t < weights.config.vocab:
            raise DomainError(f"token id {t} out of range for vocab {weights.config.vocab}")
    idx = torch.tensor(ids, dtype=torch.long, device=weights.embedding.device)
    return weights.embedding.index_select(0, idx)


def _positions_tensor(positions, device) -> torch.Tensor:
    if isinstance(positions, torch.Tensor):
        return positions.to(device=device, dtype=torch.int64)
    return torch.tensor(list(positions), dtype=torch.int64, device=device)


def project_raw(x: torch.Tensor, lw: LayerWeights, cfg: ModelConfig):
    """RMSNorm -> Q/K/V projections, before RoPE: ([rows, H, hd] x 3), attention dtype."""
    H, hd = cfg.heads, cfg.head_dim
    xn = _rms_norm(x, lw.attn_gain)
    rows = x.shape[0]
    dt = default_dtype()
    return tuple((xn @ w).view(rows, H, hd).to(dt).contiguous() for w in (lw.wq, lw.wk, lw.wv))


def project_qkv(x: torch.Tensor, lw: LayerWeights, cfg: ModelConfig, positions):
    """RMSNorm -> Q/K/V projections -> RoPE on q and k: ([rows, H, hd] x 3), attention dtype."""
    q, k, v = project_raw(x, lw, cfg)
    pos = _positions_tensor(positions, x.device)
    if pos.numel() != x.shape[0]:
        raise ConfigError(f"{pos.numel()} positions for {x.shape[0]} rows")
    return ops.rope(q, pos, cfg.rope_theta), ops.rope(k, pos, cfg.rope_theta), v


def finish_layer(x: torch.Tensor, att: torch.Tensor, lw: LayerWeights) -> torch.Tensor:
    """Residual + output projection + SiLU FFN (ss/toy_model.py:164-166)."""
    x = x + att.reshape(x.shape[0], -1).float() @ lw.wo
    xn2 = _rms_norm(x, lw.ffn_gain)
    return x + _silu(xn2 @ lw.w1) @ lw.w2


def layer_step_all(x: torch.Tensor, lw: LayerWeights, cfg: ModelConfig, positions,
                   attend_all: AttendAllFn) -> torch.Tensor:
    """One layer with all heads' attention in one call (the batched B200 form)."""
    q, k, v = project_qkv(x, lw, cfg, positions)
    return finish_layer(x, attend_all(q, k, v), lw)


def layer_step(x: torch.Tensor, lw: LayerWeights, cfg: ModelConfig, positions,
               attend: AttendFn) -> torch.Tensor:
    """Reference-compatible layer: attend(h, q_h, k_h, v_h) once per head (ss/toy_model.py:141-166)."""

    def per_head(q, k, v):
        return torch.stack([attend(h, q[:, h], k[:, h], v[:, h]) for h in range(cfg.heads)], dim=1)

    return layer_step_all(x, lw, cfg, positions, per_head)


def logits_from(weights: ModelWeights, x: torch.Tensor) -> torch.Tensor:
    """Tied output projection (ss/toy_model.py:169-171)."""
    return _rms_norm(x, weights.final_gain) @ weights.embedding.T


def forward_global(weights: ModelWeights, tokens) -> torch.Tensor:
    """Plain causal forward over positions 0..n-1 (ss/toy_model.py:174-184)."""
    x = embed(weights, tokens)
    n = x.shape[0]

    def attend_all(q, k, v):
        out, _ = ops.phase1_fwd(q, k, v, [0, n], out_dtype=torch.float32)
        return out

    for lw in weights.layers:
        x = layer_step_all(x, lw, weights.config, range(n), attend_all)
    return logits_from(weights, x)


def greedy_decode_global(weights: ModelWeights, tokens, n_steps: int) -> list[int]:
    """Full re-encode per step, argmax with lowest-id ties (ss/toy_model.py:187-196)."""
    cur = list(tokens)
    out = []
    for _ in range(n_steps):
        t = int(torch.argmax(forward_global(weights, cur)[-1]))
        out.append(t)
        cur.append(t)
    return out
