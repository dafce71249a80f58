"""Precision switch, RoPE config and the splitmix64 stream — host side of the
numerics substrate (reference: ss/numerics.py).

Device tensors replace the reference's Tensor2D.  The build-wide precision is
"float32" (the reference default, served by the fp32 check-mode kernels) or
"bfloat16" (production: tcgen05 tensor-core phase 1, bf16 paged KV).  The
reference's "float64" oracle mode has no device path and is rejected.
"""

from __future__ import annotations

from contextlib import contextmanager
from dataclasses import dataclass

import numpy as np
import torch

from .errors import ConfigError, DomainError

_DTYPES = {"float32": torch.float32, "bfloat16": torch.bfloat16}
_default = torch.float32


def default_dtype() -> torch.dtype:
    """Current build-wide compute dtype for attention inputs / KV caches."""
    return _default


def set_default_dtype(dtype) -> None:
    """Switch the build-wide precision ("float32" check mode or "bfloat16")."""
    global _default
    if isinstance(dtype, torch.dtype):
        if dtype not in _DTYPES.values():
            raise ConfigError(f"unsupported scalar dtype {dtype}; use float32 or bfloat16")
        _default = dtype
        return
    name = str(np.dtype(dtype).name) if dtype not in _DTYPES else dtype
    if name not in _DTYPES:
        raise ConfigError(f"unsupported scalar dtype {dtype}; use float32 or bfloat16 "
                          "(float64 oracle mode has no device path)")
    _default = _DTYPES[name]


@contextmanager
def precision(dtype):
    """Temporarily run under a different build-wide precision (ss/numerics.py:36-44)."""
    prev = _default
    set_default_dtype(dtype)
    try:
        yield
    finally:
        set_default_dtype(prev)


@dataclass(frozen=True)
class RopeConfig:
    """Rotary parameters for one head (ss/numerics.py:109-120)."""

    head_dim: int
    theta_base: float = 10000.0

    def __post_init__(self):
        if self.head_dim < 2 or self.head_dim % 2 != 0:
            raise ConfigError(f"rope head_dim must be even and >= 2, got {self.head_dim}")
        if self.theta_base <= 0:
            raise ConfigError(f"rope theta_base must be positive, got {self.theta_base}")


def rope_apply(x, positions, cfg: RopeConfig) -> torch.Tensor:
    """Rotate adjacent coordinate pairs of each row by its position's angles
    (ss/numerics.py:161-180): pair i of a row at position p turns by p * theta^(-2i/d), angles
    in fp64.  x: one head's [rows, head_dim] (numpy / Tensor2D / torch); returns a device
    tensor in the build precision (star_rope)."""
    from . import ops
    from .blocking import _as_device_2d
    from .errors import ShapeError

    t = _as_device_2d(x)
    if t.shape[1] != cfg.head_dim:
        raise ShapeError(f"rope input has {t.shape[1]} cols, config head_dim {cfg.head_dim}")
    pos = torch.as_tensor(np.asarray(positions, dtype=np.int64).reshape(-1)).to(t.device)
    if pos.numel() != t.shape[0]:
        raise ShapeError(f"{pos.numel()} positions for {t.shape[0]} rows")
    if t.shape[0] == 0:
        return t.clone()
    return ops.rope(t.contiguous().view(t.shape[0], 1, t.shape[1]), pos,
                    cfg.theta_base).view(t.shape)


_M64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


def _mix(z: int) -> int:
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & _M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


class Prng:
    """Counter-based splitmix64 stream (ss/numerics.py:199-252).

    Draw i (1-based) is mix64(seed + i*golden).  Small draws (token ids, anchor
    positions) run on the host; bulk tensors come from the device kernel
    `prng_fill`, which consumes the same counter range.
    """

    def __init__(self, seed: int):
        self.seed = int(seed) & _M64
        self._count = 0

    def next_u64(self) -> int:
        self._count += 1
        return _mix((self.seed + self._count * _GOLDEN) & _M64)

    def next_float(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def randint_below(self, n: int) -> int:
        if n <= 0:
            raise DomainError(f"randint_below needs n >= 1, got {n}")
        return self.next_u64() % n

    def shuffle(self, items) -> list:
        out = list(items)
        for i in range(len(out) - 1, 0, -1):
            j = self.randint_below(i + 1)
            out[i], out[j] = out[j], out[i]
        return out

    def sample_sorted(self, n: int, k: int) -> list[int]:
        if k > n:
            raise DomainError(f"cannot sample {k} distinct values from range {n}")
        chosen: set[int] = set()
        for j in range(n - k, n):
            t = self.randint_below(j + 1)
            chosen.add(t if t not in chosen else j)
        return sorted(chosen)

    def take(self, n: int) -> int:
        """Reserve n draws; returns the 1-based index of the first (for device fills)."""
        first = self._count + 1
        self._count += n
        return first


def prng_fill(prng: Prng, rows: int, cols: int, scale: float, dtype=None, device="cuda"):
    """Device tensor of uniforms in [-scale, scale] drawn from `prng` (ss/numerics.py:255-263)."""
    from . import ops

    if scale <= 0:
        raise DomainError(f"prng_fill scale must be positive, got {scale}")
    first = prng.take(rows * cols)
    return ops.prng_fill((rows, cols), prng.seed, first, scale, dtype or torch.float32, device)
