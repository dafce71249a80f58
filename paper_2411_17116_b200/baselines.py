"""Analytic cost models and the divergence metric (reference: ss/baselines.py).

star_model gives the algorithmic phase-1 score-pair count that bench.py turns
into the tensor-core roofline (pairs x Hq x 4d FLOP).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .errors import ConfigError, ShapeError


@dataclass(frozen=True)
class FlopReport:
    """Score pairs and communicated scalars split by phase (ss/baselines.py:59-93)."""

    phase1_pairs: int
    phase2_pairs: int
    phase1_comm: int
    phase2_comm: int

    def __post_init__(self):
        for name in ("phase1_pairs", "phase2_pairs", "phase1_comm", "phase2_comm"):
            if getattr(self, name) < 0:
                raise ConfigError(f"{name} cannot be negative")

    @property
    def score_pairs(self) -> int:
        return self.phase1_pairs + self.phase2_pairs

    @property
    def comm_scalars(self) -> int:
        return self.phase1_comm + self.phase2_comm

    def to_json(self) -> dict:
        return {"score_pairs": self.score_pairs, "comm_scalars": self.comm_scalars,
                "phase1_pairs": self.phase1_pairs, "phase2_pairs": self.phase2_pairs,
                "phase1_comm": self.phase1_comm, "phase2_comm": self.phase2_comm}


def _query_phase_pairs(L: int, l_q: int, n_generated: int) -> int:
    # closed forms of sum_{i<l_q}(L+i+1) and sum_{t<n}(L+l_q+t+1)
    return l_q * (L + 1) + l_q * (l_q - 1) // 2 + n_generated * (L + l_q + 1) + \
        n_generated * (n_generated - 1) // 2


def ring_model(L: int, H: int, d: int, heads: int = 1) -> FlopReport:
    """Analytic ring baseline (ss/baselines.py:103-121)."""
    if H < 1:
        raise ConfigError(f"ring needs >= 1 host, got {H}")
    if L < 1:
        raise ConfigError(f"ring needs L >= 1, got {L}")
    shard = -(-L // H)
    return FlopReport(L * (L + 1) // 2, 0, H * (H - 1) * 2 * shard * d * heads, 0)


def star_model(L: int, b: int, anchor_len: int | None = None, d: int = 0, heads: int = 1,
               l_q: int = 0, n_generated: int = 0, hosts: int | None = None) -> FlopReport:
    """Blockwise causal pairs + aggregation traffic (ss/baselines.py:124-160)."""
    if b < 1 or L < 1:
        raise ConfigError(f"star model needs L >= 1 and b >= 1, got L={L}, b={b}")
    if b > L:
        raise ConfigError(f"block size {b} exceeds context length {L}")
    a = b if anchor_len is None else anchor_len
    if a > b:
        raise ConfigError(f"anchor_len {a} exceeds block size {b}")
    n = -(-L // b)
    pairs = 0
    for i in range(n):
        m = min(b, L - i * b) + (a if i else 0)
        pairs += m * (m + 1) // 2
    H = n if hosts is None else hosts
    comm = (H - 1) * (l_q + n_generated) * (d + 1) * heads
    return FlopReport(pairs, _query_phase_pairs(L, l_q, n_generated), 0, comm)


def global_pairs(L: int, l_q: int = 0, n_generated: int = 0) -> int:
    return L * (L + 1) // 2 + _query_phase_pairs(L, l_q, n_generated)


@dataclass(frozen=True)
class DivergenceReport:
    max_abs: float
    mean_abs: float
    cosine_per_row_min: float

    def to_json(self) -> dict:
        return {"max_abs": self.max_abs, "mean_abs": self.mean_abs,
                "cosine_per_row_min": self.cosine_per_row_min}


def divergence(a: torch.Tensor, b: torch.Tensor) -> DivergenceReport:
    """Elementwise gap between two same-shape outputs (ss/baselines.py:168-203)."""
    if tuple(a.shape) != tuple(b.shape):
        raise ShapeError(f"divergence of mismatched shapes {tuple(a.shape)} vs {tuple(b.shape)}")
    aa, bb = a.double(), b.double()
    diff = (aa - bb).abs()
    na, nb = aa.norm(dim=1), bb.norm(dim=1)
    cos = (aa * bb).sum(1) / (na * nb)
    cos = torch.where((na == 0) & (nb == 0), torch.ones_like(cos),
                      torch.where((na == 0) | (nb == 0), torch.zeros_like(cos), cos))
    return DivergenceReport(float(diff.max()), float(diff.mean()), float(cos.min()))
