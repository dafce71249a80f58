"""Context partitioning, anchor-augmented blocks and the paged per-host KV cache.

Layout contract of the reference (ss/blocking.py): partition / AnchorSpec /
augment / AugmentedBlock are restated bit-exactly (tests/test_layout.py pins
them to the reference's golden vectors).  The KV cache is B200-native: one
paged pool per host, [layers][num_pages, hkv, page_size, head_dim] in HBM,
addressed through an int32 page table; `KVCache` is a per-(layer, head)
channel view onto it, so `Host.channels[li*heads + h]` reads like the
reference's list of caches.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .errors import ConfigError, ShapeError
from .numerics import Prng, default_dtype

CONTENT_MODES = (
    "first_block",
    "none",
    "previous_block",
    "random_tokens",
    "shuffled_first_block",
    "constant_token",
)
POSITION_MODES = ("first_block", "previous_block", "random_sampled")


@dataclass(frozen=True)
class BlockPlan:
    """Partition of [0, L) into contiguous blocks, each owned by one host (ss/blocking.py:31-46)."""

    context_len: int
    block_size: int
    num_blocks: int
    num_hosts: int
    host_assignment: tuple[int, ...]

    def block_span(self, i: int) -> tuple[int, int]:
        start = i * self.block_size
        return start, min(start + self.block_size, self.context_len)

    def blocks_of(self, host: int) -> list[int]:
        return [i for i, h in enumerate(self.host_assignment) if h == host]


def partition(L: int, b: int, num_hosts: int | None = None, allow_idle: bool = False) -> BlockPlan:
    """ceil(L/b) blocks, contiguous balanced runs: block i -> min(i*H//n, H-1) (ss/blocking.py:49-69)."""
    if L < 1:
        raise ConfigError(f"context length must be >= 1, got {L}")
    if b < 1:
        raise ConfigError(f"block size must be >= 1, got {b}")
    n = -(-L // b)
    H = n if num_hosts is None else num_hosts
    if H < 1:
        raise ConfigError(f"host count must be >= 1, got {H}")
    if H > n and not allow_idle:
        raise ConfigError(f"{H} hosts for {n} blocks; pass allow_idle to permit")
    return BlockPlan(L, b, n, H, tuple(min(i * H // n, H - 1) for i in range(n)))


@dataclass(frozen=True)
class AnchorSpec:
    """Anchor content / position strategy (ss/blocking.py:72-118)."""

    content_mode: str = "first_block"
    position_mode: str = "first_block"
    anchor_len: int | None = None
    constant_token_id: int = 0
    token_range: int = 256

    def __post_init__(self):
        if self.content_mode not in CONTENT_MODES:
            raise ConfigError(f"unknown anchor content_mode {self.content_mode!r}")
        if self.position_mode not in POSITION_MODES:
            raise ConfigError(f"unknown anchor position_mode {self.position_mode!r}")
        if self.anchor_len is not None and self.anchor_len < 1:
            raise ConfigError(f"anchor_len must be >= 1, got {self.anchor_len}")
        if self.token_range < 1:
            raise ConfigError(f"token_range must be >= 1, got {self.token_range}")

    def to_config(self) -> dict:
        return {"content_mode": self.content_mode, "position_mode": self.position_mode,
                "anchor_len": self.anchor_len, "constant_token_id": self.constant_token_id,
                "token_range": self.token_range}

    @classmethod
    def from_config(cls, doc: dict) -> "AnchorSpec":
        for key in doc:
            if key not in ("content_mode", "position_mode", "anchor_len", "constant_token_id",
                           "token_range"):
                raise ConfigError(f"unknown anchor field '{key}'")
        return cls(**doc)


@dataclass(frozen=True)
class AugmentedBlock:
    """One block plus its anchor prefix with explicit position ids (ss/blocking.py:121-142)."""

    token_ids: tuple[int, ...]
    position_ids: tuple[int, ...]
    anchor_prefix_len: int
    block_index: int

    def __post_init__(self):
        if len(self.token_ids) != len(self.position_ids):
            raise ShapeError(f"{len(self.token_ids)} tokens vs {len(self.position_ids)} positions")

    @property
    def own_len(self) -> int:
        return len(self.token_ids) - self.anchor_prefix_len

    @property
    def own_positions(self) -> tuple[int, ...]:
        return self.position_ids[self.anchor_prefix_len:]


def _anchor_tokens(spec: AnchorSpec, tokens, start: int, a_len: int, prng: Prng):
    mode = spec.content_mode
    if mode == "first_block":
        return tuple(tokens[:a_len])
    if mode == "previous_block":
        return tuple(tokens[start - a_len:start])
    if mode == "shuffled_first_block":
        return tuple(prng.shuffle(tokens[:a_len]))
    if mode == "random_tokens":
        return tuple(prng.randint_below(spec.token_range) for _ in range(a_len))
    if mode == "constant_token":
        return (spec.constant_token_id,) * a_len
    raise ConfigError(f"unsupported content_mode {mode!r}")


def _anchor_positions(spec: AnchorSpec, start: int, a_len: int, prng: Prng):
    mode = spec.position_mode
    if mode == "first_block":
        return tuple(range(a_len))
    if mode == "previous_block":
        return tuple(range(start - a_len, start))
    if mode == "random_sampled":
        return tuple(prng.sample_sorted(start, a_len))
    raise ConfigError(f"unsupported position_mode {mode!r}")


def augment(plan: BlockPlan, tokens, spec: AnchorSpec, prng: Prng | None = None) -> list[AugmentedBlock]:
    """Anchor-augmented view of every block (ss/blocking.py:206-236)."""
    tokens = list(tokens)
    if len(tokens) != plan.context_len:
        raise ConfigError(f"{len(tokens)} tokens for a plan covering {plan.context_len}")
    a_len = plan.block_size if spec.anchor_len is None else spec.anchor_len
    if a_len > plan.block_size:
        raise ConfigError(f"anchor_len {a_len} exceeds block size {plan.block_size}")
    prng = prng or Prng(0)
    blocks = []
    for i in range(plan.num_blocks):
        start, end = plan.block_span(i)
        own, own_pos = tuple(tokens[start:end]), tuple(range(start, end))
        if i == 0 or spec.content_mode == "none":
            blocks.append(AugmentedBlock(own, own_pos, 0, i))
            continue
        ank = _anchor_tokens(spec, tokens, start, a_len, prng)
        ank_pos = _anchor_positions(spec, start, a_len, prng)
        blocks.append(AugmentedBlock(ank + own, ank_pos + own_pos, a_len, i))
    return blocks


def sparsity_pattern(plan: BlockPlan, spec: AnchorSpec) -> np.ndarray:
    """Block-granular attention mask, n context rows + the query row (ss/blocking.py:268-285)."""
    n = plan.num_blocks
    pat = np.zeros((n + 1, n + 1), dtype=bool)
    for i in range(n):
        pat[i, i] = True
        if i and spec.content_mode in ("first_block", "shuffled_first_block"):
            pat[i, 0] = True
        elif i and spec.content_mode == "previous_block":
            pat[i, i - 1] = True
    pat[n, :] = True
    return pat


# ---------------------------------------------------------------------------- paged KV
class PagedKVPool:
    """One host's KV cache for every layer, paged in HBM.

    k/v: [layers, num_pages, hkv, page_size, head_dim]; logical row r of every
    (layer, head) lives in page page_table[r // page_size], slot r % page_size.
    Rows are appended in place (the reference copies the whole cache on each
    append, ss/blocking.py:161-170).  `layer_rows[li]` counts the rows layer li
    holds; `positions` are the global position ids of the rows, shared by all
    channels (ss/sim.py:151-174).
    """

    def __init__(self, layers: int, hkv: int, head_dim: int, capacity_rows: int = 0,
                 page_size: int = 128, dtype=None, device="cuda"):
        if page_size % 64:
            raise ConfigError(f"page_size must be a multiple of 64, got {page_size}")
        self.layers, self.hkv, self.head_dim, self.page_size = layers, hkv, head_dim, page_size
        self.dtype = dtype or default_dtype()
        self.device = torch.device(device)
        self.layer_rows = [0] * layers
        self.positions: list[int] = []
        self.k = self.v = None
        self.page_table = None
        # device mirror of layer_rows: the K2 kv_len argument and the row counter of
        # append_rope (graph-safe: a captured decode step advances it on the device)
        self.kv_len_dev = torch.zeros(layers, dtype=torch.int32, device=self.device)
        self._workspace = None
        self._alloc(max(capacity_rows, page_size))

    def _alloc(self, rows: int) -> None:
        n_pages = -(-rows // self.page_size)
        shape = (self.layers, n_pages, self.hkv, self.page_size, self.head_dim)
        k = torch.zeros(shape, dtype=self.dtype, device=self.device)
        v = torch.zeros_like(k)
        if self.k is not None:
            old = self.k.shape[1]
            k[:, :old].copy_(self.k)
            v[:, :old].copy_(self.v)
        self.k, self.v = k, v
        self.page_table = torch.arange(n_pages, dtype=torch.int32, device=self.device)

    @property
    def capacity(self) -> int:
        return self.k.shape[1] * self.page_size

    def reserve(self, rows: int, exact: bool = False) -> None:
        """Grow to at least `rows` rows (doubling, or exactly `rows` rounded to pages)."""
        if rows > self.capacity:
            self._alloc(rows if exact else max(rows, 2 * self.capacity))

    def head_view(self, layer: int, head: int):
        """One kv head of `layer` as a single-head pool: (k, v, page_table), k/v viewed as
        [num_pages * hkv, 1, page_size, d] (no copy) and the table remapped to
        page * hkv + head, so K2 streams that head's rows only (one channel of
        ss/sim.py:216-237 reads 1/hkv of the layer's bytes)."""
        n_pages = self.k.shape[1]
        shape = (n_pages * self.hkv, 1, self.page_size, self.head_dim)
        key = (n_pages, head)
        cache = getattr(self, "_head_tables", None)
        if cache is None or cache[0] is not self.page_table:
            cache = self._head_tables = (self.page_table, {})
        table = cache[1].get(key)
        if table is None:
            table = cache[1][key] = (self.page_table * self.hkv + head).to(torch.int32)
        return self.k[layer].view(shape), self.v[layer].view(shape), table

    @property
    def workspace(self):
        """This pool's K2 split workspace (one per pool, so the hosts' launches never share
        split counters and each keeps a stable shape signature)."""
        if self._workspace is None:
            self._workspace = ops.Phase2Workspace()
        return self._workspace

    def write(self, layer: int, k: torch.Tensor, v: torch.Tensor, row0: int) -> None:
        """Write k/v [n, hkv, d] at logical rows [row0, row0+n) of `layer`."""
        n = k.shape[0]
        self.reserve(row0 + n)
        ops.kv_write(k.to(self.dtype), v.to(self.dtype), self.k[layer], self.v[layer],
                     self.page_table, row0)
        if row0 + n > self.layer_rows[layer]:
            self.layer_rows[layer] = row0 + n
            self.kv_len_dev[layer:layer + 1].fill_(row0 + n)  # stream-ordered, no host copy

    def append(self, layer: int, k: torch.Tensor, v: torch.Tensor, positions) -> None:
        """Append rows to one layer (new positions are recorded by the first layer to reach them)."""
        row0 = self.layer_rows[layer]
        pos = list(positions)
        if len(pos) != k.shape[0]:
            raise ShapeError("appended keys/values/positions disagree in length")
        self.write(layer, k, v, row0)
        if row0 + len(pos) > len(self.positions):
            self.positions.extend(pos[len(self.positions) - row0:])

    def append_rope(self, layer: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                    positions: torch.Tensor, theta: float, table=None) -> torch.Tensor:
        """Graph-safe append of one step's rows (star_kv_append, one launch): RoPE of q and k
        at the device `positions`, rotated k and raw v written at the rows the device counter
        kv_len_dev[layer] names, counter advanced on the device.  Returns rotated q.
        The host mirror (layer_rows, positions) is the caller's to advance (DeviceDecoder)."""
        dt = self.dtype
        return ops.kv_append(q.to(dt).contiguous(), k.to(dt).contiguous(), v.to(dt).contiguous(),
                             positions, self.kv_len_dev[layer:layer + 1], self.k[layer],
                             self.v[layer], self.page_table, theta, table=table)

    def rows(self, layer: int) -> int:
        return self.layer_rows[layer]

    def kv_len_tensor(self, layer: int) -> torch.Tensor:
        """[1] int32 device view of layer's row count (no host->device copy per call)."""
        return self.kv_len_dev[layer:layer + 1]

    def dense(self, layer: int, head: int | None = None):
        """Materialise a layer's rows densely: ([rows, hkv, d], [rows, hkv, d]) (checks only)."""
        k, v = ops.kv_read(self.k[layer], self.v[layer], self.page_table, 0, self.layer_rows[layer])
        if head is not None:
            return k[:, head], v[:, head]
        return k, v


class KVCache:
    """Per-channel view (layer, head) of a host's paged pool (reference: ss/blocking.py:145-179).

    Construct either from dense keys/values (like the reference) — which
    creates a private one-layer, one-head pool — or as a view onto a host pool.
    `append` on a dense-constructed cache returns a NEW cache and leaves this one unchanged
    (the reference's value semantics, ss/blocking.py:161-170); on a host-pool view it grows
    the host's pool in place and returns self (the protocol's query-host append).
    """

    def __init__(self, keys=None, values=None, positions=(), host: int = 0, *,
                 pool: PagedKVPool | None = None, layer: int = 0, head: int = 0):
        self.host = host
        self._private = pool is None
        if pool is None:
            k = _as_device_2d(keys)
            vv = _as_device_2d(values)
            pos = tuple(int(p) for p in positions)
            if not (k.shape[0] == vv.shape[0] == len(pos)):
                raise ShapeError(f"cache rows disagree: keys {k.shape[0]}, values {vv.shape[0]}, "
                                 f"positions {len(pos)}")
            if k.shape[1] != vv.shape[1]:
                raise ShapeError("keys and values must share head_dim")
            pool = PagedKVPool(1, 1, k.shape[1], max(k.shape[0], 1), page_size=64,
                               device=k.device)
            if k.shape[0]:
                pool.append(0, k.unsqueeze(1), vv.unsqueeze(1), pos)
            layer, head = 0, 0
        self.pool, self.layer, self.head = pool, layer, head

    @property
    def rows(self) -> int:
        return self.pool.rows(self.layer)

    @property
    def positions(self) -> tuple[int, ...]:
        return tuple(self.pool.positions[: self.rows])

    @property
    def keys(self) -> torch.Tensor:
        return self.pool.dense(self.layer, self.head)[0]

    @property
    def values(self) -> torch.Tensor:
        return self.pool.dense(self.layer, self.head)[1]

    def append(self, keys, values, positions) -> "KVCache":
        k, v = _as_device_2d(keys), _as_device_2d(values)
        pos = tuple(positions)
        if k.shape[0] != v.shape[0] or k.shape[0] != len(pos):
            raise ShapeError("appended keys/values/positions disagree in length")
        if self._private:
            if self.rows and k.shape[1] != self.pool.head_dim:
                raise ShapeError("appended keys must share head_dim")
            keys = torch.cat([self.keys, k]) if self.rows else k
            values = torch.cat([self.values, v]) if self.rows else v
            return KVCache(keys, values, self.positions + tuple(int(p) for p in pos), self.host)
        if self.pool.hkv != 1:
            raise ShapeError("append through a multi-head pool goes through PagedKVPool.append")
        self.pool.append(self.layer, k.unsqueeze(1), v.unsqueeze(1), pos)
        return self

    @classmethod
    def concat(cls, caches: list["KVCache"], host: int) -> "KVCache":
        keys = torch.cat([c.keys for c in caches])
        values = torch.cat([c.values for c in caches])
        return cls(keys, values, sum((c.positions for c in caches), ()), host)


def _as_device_2d(x) -> torch.Tensor:
    """numpy / reference Tensor2D / torch -> 2-D CUDA tensor in the build precision."""
    if hasattr(x, "a") and not isinstance(x, torch.Tensor):  # reference Tensor2D
        x = x.a
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x))
    if t.dim() != 2:
        raise ShapeError(f"expected a 2-D matrix, got shape {tuple(t.shape)}")
    if not t.is_cuda:
        t = t.cuda()
    return t.to(default_dtype())


def encode_block(block: AugmentedBlock, embedding, wq, wk, wv, rope, host: int = 0) -> KVCache:
    """One attention channel over an augmented block, keeping only the own rows' K/V
    (ss/blocking.py:239-265).  The whole block (anchor rows included) runs as queries
    through the causal block encode (K1 in bf16, the fp32 check-mode kernel otherwise); the
    outputs are computed and dropped as in the reference.  Returns KVCache(rotated k[a:],
    v[a:], own positions, host)."""
    from .attention import causal_attention
    from .errors import DomainError
    from .numerics import rope_apply

    emb = _as_device_2d(embedding).float()
    for t in block.token_ids:
        if not 0 <= t < emb.shape[0]:
            raise DomainError(f"token id {t} outside embedding table of {emb.shape[0]}")
    idx = torch.tensor(block.token_ids, dtype=torch.long, device=emb.device)
    x = emb.index_select(0, idx)
    dt = default_dtype()
    proj = [(x @ _as_device_2d(w).float()).to(dt) for w in (wq, wk, wv)]
    q = rope_apply(proj[0], block.position_ids, rope)
    k = rope_apply(proj[1], block.position_ids, rope)
    v = proj[2]
    causal_attention(q, k, v)  # anchor-row outputs are computed, then dropped
    lo = block.anchor_prefix_len
    return KVCache(k[lo:], v[lo:], block.own_positions, host)
