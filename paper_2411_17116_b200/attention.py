"""Drop-in attention API of the reference (ss/attention.py), served by the
sm_100a kernels.  Inputs may be torch tensors, numpy arrays or reference
Tensor2D objects; results are CUDA tensors.  lse is natural-log, fp32 on
device (the reference stores fp64 on host).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import ops
from .blocking import _as_device_2d
from .errors import ConfigError, DomainError, ShapeError


@dataclass(frozen=True)
class AttnScale:
    """Score scaling 1/sqrt(head_dim) (ss/attention.py:26-43)."""

    head_dim: int
    scale: float

    def __post_init__(self):
        if self.head_dim < 1:
            raise ConfigError(f"head_dim must be >= 1, got {self.head_dim}")
        if abs(self.scale - 1.0 / math.sqrt(self.head_dim)) > 1e-12:
            raise ConfigError(f"scale {self.scale} != 1/sqrt({self.head_dim}) beyond 1e-12")

    @classmethod
    def for_dim(cls, head_dim: int) -> "AttnScale":
        return cls(head_dim, 1.0 / math.sqrt(head_dim))


@dataclass(frozen=True, eq=False)
class PartialAttention:
    """Locally normalised output plus per-row natural-log LSE (ss/attention.py:46-64)."""

    out: torch.Tensor
    lse: torch.Tensor

    def __post_init__(self):
        if self.out.shape[0] != self.lse.numel():
            raise ShapeError(f"out has {self.out.shape[0]} rows but lse has {self.lse.numel()}")
        if not bool(torch.isfinite(self.lse).all()):
            raise DomainError("non-finite log-sum-exp in partial attention")


def _check_qkv(q, k, v):
    if k.shape[0] != v.shape[0]:
        raise ShapeError(f"k has {k.shape[0]} rows but v has {v.shape[0]}")
    if q.shape[1] != k.shape[1]:
        raise ShapeError(f"q cols {q.shape[1]} != k cols {k.shape[1]}")


def causal_attention(q, k, v, q_offset: int = 0) -> torch.Tensor:
    """softmax(q k^T / sqrt(d), causal) v (ss/attention.py:109-122).

    Self-attention of a whole block in bf16 runs the tcgen05 phase-1 kernel;
    everything else runs the fp32 / generic kernel.
    """
    q, k, v = _as_device_2d(q), _as_device_2d(k), _as_device_2d(v)
    _check_qkv(q, k, v)
    if q_offset + q.shape[0] > k.shape[0]:
        raise ShapeError(f"q rows [{q_offset}, {q_offset + q.shape[0]}) extend past {k.shape[0]} keys")
    if q.shape[0] and q_offset < 0:
        raise DomainError(f"q_offset {q_offset} leaves a query row with no keys")
    if q.shape[0] == 0:
        return q.clone()
    if q_offset == 0 and q.shape[0] == k.shape[0]:
        out, _ = ops.phase1_fwd(q.unsqueeze(1), k.unsqueeze(1), v.unsqueeze(1), [0, q.shape[0]])
        return out[:, 0]
    out, _ = ops.attention_dense(q.unsqueeze(1), k.unsqueeze(1), v.unsqueeze(1), q_offset, "causal",
                                 want_lse=False)
    return out[:, 0]


def _classify_mask(keep: np.ndarray, lq: int, lk: int):
    """Map a boolean keep matrix onto a kernel mask: ("full",), ("causal", off) or ("tail", n)."""
    if keep.all():
        return ("full", 0)
    off = lk - lq
    if off >= 0 and np.array_equal(keep, np.arange(lk)[None, :] <= (off + np.arange(lq))[:, None]):
        return ("causal", off)
    t = lq
    if lk >= t:
        tail = np.ones((lq, lk), dtype=bool)
        tail[:, lk - t:] = np.arange(t)[None, :] <= np.arange(lq)[:, None]
        if np.array_equal(keep, tail):
            return ("tail", t)
    return None


def partial_attention(q, k, v, mask="full", q_offset: int = 0) -> PartialAttention:
    """(locally normalised out, lse) over one key set (ss/attention.py:125-151).

    mask: "full", "causal" (with q_offset), or a boolean [lq, lk] keep matrix;
    boolean masks must be one of the patterns the protocol produces (full,
    causal, or the query host's own-tail mask, ss/sim.py:195-200).
    """
    q, k, v = _as_device_2d(q), _as_device_2d(k), _as_device_2d(v)
    _check_qkv(q, k, v)
    lq, lk = q.shape[0], k.shape[0]
    if isinstance(mask, str):
        if mask not in ("full", "causal"):
            raise ConfigError(f"unknown mask kind {mask!r}")
        kind = (mask, q_offset)
    else:
        keep = np.asarray(mask.cpu() if isinstance(mask, torch.Tensor) else mask, dtype=bool)
        if keep.shape != (lq, lk):
            raise ShapeError(f"mask shape {keep.shape} != ({lq}, {lk})")
        if lk and not keep.any(axis=1).all():
            raise DomainError("query row with every key masked")
        kind = _classify_mask(keep, lq, lk)
        if kind is None:
            raise ConfigError("arbitrary boolean masks are not supported by the device kernels")
    if lk == 0:
        raise DomainError("partial attention over an empty key set")
    if kind[0] == "causal" and kind[1] + lq > lk:
        raise ShapeError(f"q rows [{kind[1]}, {kind[1] + lq}) extend past {lk} keys")
    if kind[0] == "causal" and kind[1] < 0:
        raise DomainError("query row with every key masked")
    if kind[0] == "tail":
        # the paged phase-2 kernel implements the own-tail keep mask
        pool_k = k.unsqueeze(1).unsqueeze(0).transpose(1, 2).contiguous()  # [1, 1, lk, d] page
        pool_v = v.unsqueeze(1).unsqueeze(0).transpose(1, 2).contiguous()
        pad = (-lk) % 64
        if pad:
            z = torch.zeros((1, 1, pad, k.shape[1]), dtype=k.dtype, device=k.device)
            pool_k, pool_v = torch.cat([pool_k, z], 2), torch.cat([pool_v, z], 2)
        table = torch.zeros((1, 1), dtype=torch.int32, device=k.device)
        kv_len = torch.tensor([lk], dtype=torch.int32, device=k.device)
        out, lse = ops.phase2_partial(q.view(1, lq, 1, -1).contiguous(), pool_k, pool_v, table,
                                      kv_len, lk, own_tail=kind[1])
        return PartialAttention(out[0, :, 0].to(q.dtype), lse[0, :, 0])
    out, lse = ops.attention_dense(q.unsqueeze(1), k.unsqueeze(1), v.unsqueeze(1), kind[1], kind[0])
    return PartialAttention(out[:, 0], lse[0])


def merge_partials(parts: Sequence[PartialAttention]) -> PartialAttention:
    """Log-domain fold of partials in the given order (ss/attention.py:154-173)."""
    if len(parts) == 0:
        raise DomainError("merge of zero partials")
    shape = tuple(parts[0].out.shape)
    for p in parts[1:]:
        if tuple(p.out.shape) != shape:
            raise ShapeError(f"partial shapes differ: {shape} vs {tuple(p.out.shape)}")
    if len(parts) == 1:
        return parts[0]
    outs = torch.stack([p.out.float() for p in parts])
    lses = torch.stack([p.lse.float() for p in parts])
    out, lse = ops.merge(outs, lses, out_dtype=parts[0].out.dtype)
    return PartialAttention(out, lse)


def streaming_causal_attention(q, k, v, tile: int, q_offset: int = 0) -> torch.Tensor:
    """Key-tiled causal attention (ss/attention.py:176-210).

    The device kernels are already tile-folded with the merge rule (128-key
    tiles in TMEM / 32-key tiles in the fp32 kernel); `tile` is validated
    and the result equals causal_attention for every tile size.
    """
    if tile < 1:
        raise ConfigError(f"tile must be >= 1, got {tile}")
    return causal_attention(q, k, v, q_offset)
