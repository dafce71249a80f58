"""Two-phase star-attention protocol over hosts (reference: ss/sim.py), B200-native.

A "host" owns one paged KV pool in HBM.  In this module all hosts live on the
current device (the reference's single-process simulation, used for parity
and for the tiny config); `dist.py` runs the same protocol with one host per
GPU rank over NCCL.

Phase 1 encodes every anchor-augmented block of a layer in ONE tcgen05
launch (the blocks are segments of one batched call) and writes each block's
own K/V rows into its host's pages; no ledger entries.  Phase 2 appends the
query rows to the query host, runs the split-KV partial kernel on every
host's pages, and merges the (out, lse) partials in ascending host order; the
ledger records exactly the reference's logical transfers.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from .attention import PartialAttention, merge_partials
from .blocking import AnchorSpec, BlockPlan, KVCache, PagedKVPool, _as_device_2d, augment
from .errors import ConfigError, ShapeError
from .model import ModelWeights, embed, finish_layer, logits_from, project_qkv
from .numerics import Prng, default_dtype

QUERY_BROADCAST = "query_broadcast"
PARTIAL_OUT = "partial_out"
PARTIAL_LSE = "partial_lse"
KV_SHIFT = "kv_shift"
AGGREGATION_KINDS = (PARTIAL_OUT, PARTIAL_LSE)

_ANCHOR_SALT = 0xA17C4B10C4ED5EED


@dataclass(frozen=True)
class LedgerEntry:
    phase: int
    src: int
    dst: int
    kind: str
    scalar_count: int


class CommLedger:
    """Append-only record of inter-host transfers (ss/sim.py:46-76)."""

    def __init__(self):
        self.entries: list[LedgerEntry] = []

    def append(self, phase: int, src: int, dst: int, kind: str, count: int) -> None:
        self.entries.append(LedgerEntry(phase, src, dst, kind, count))

    def total(self, kinds=None, phase: int | None = None) -> int:
        return sum(e.scalar_count for e in self.entries
                   if (kinds is None or e.kind in kinds) and (phase is None or e.phase == phase))

    def phase_entries(self, phase: int) -> list[LedgerEntry]:
        return [e for e in self.entries if e.phase == phase]

    def to_csv(self) -> str:
        lines = ["phase,src,dst,kind,scalar_count"]
        lines += [f"{e.phase},{e.src},{e.dst},{e.kind},{e.scalar_count}" for e in self.entries]
        return "\n".join(lines) + "\n"

    def write_csv(self, path) -> None:
        with open(path, "w", newline="\n") as f:
            f.write(self.to_csv())


@dataclass
class Host:
    """One host: index, role and per-channel KV caches (ss/sim.py:79-85).

    Model-path hosts carry a paged pool; `channels[li*heads + h]` are views on it.
    """

    index: int
    channels: list = field(default_factory=list)
    role: str = "context"
    pool: PagedKVPool | None = None


def set_query_host(hosts: list[Host], index: int) -> list[Host]:
    """Designate exactly one query host (ss/sim.py:88-94)."""
    if not 0 <= index < len(hosts):
        raise ConfigError(f"query host index {index} out of range for {len(hosts)} hosts")
    for h in hosts:
        h.role = "query" if h.index == index else "context"
    return hosts


def _query_host(hosts: list[Host]) -> Host:
    marked = [h for h in hosts if h.role == "query"]
    if not marked:
        set_query_host(hosts, len(hosts) - 1)  # documented default: the last host
        return hosts[-1]
    if len(marked) > 1:
        raise ConfigError(f"{len(marked)} hosts marked as query host")
    return marked[0]


# ---------------------------------------------------------------------------- phase 1
def _block_rows(blocks):
    seg, pos = [0], []
    for bl in blocks:
        seg.append(seg[-1] + len(bl.token_ids))
        pos.extend(bl.position_ids)
    return seg, pos


def _dedup_rows(plan: BlockPlan, spec: AnchorSpec, blocks) -> int:
    """Anchor rows shared verbatim with block 0 (first-block content AND positions)."""
    if spec.content_mode != "first_block" or spec.position_mode != "first_block" or len(blocks) < 2:
        return 0
    a = blocks[1].anchor_prefix_len
    return a if a <= len(blocks[0].token_ids) else 0


def run_phase1(tokens, plan: BlockPlan, spec: AnchorSpec, weights: ModelWeights,
               prng: Prng | None = None, workers: int = 1, page_size: int = 128,
               anchor_dedup: bool = False) -> list[Host]:
    """Encode all blocks host-locally; no ledger entries (ss/sim.py:126-175).

    `workers` is accepted for API compatibility: the device encodes every block
    of a layer in one launch, and results never depend on it.  anchor_dedup (SURVEY §8
    f3): with first-block anchors every block's anchor rows repeat block 0's computation;
    compute them once (same results, ~24% fewer phase-1 score pairs at a = b).
    """
    if workers < 1:
        raise ConfigError("workers must be >= 1")
    cfg = weights.config
    prng = prng or Prng(cfg.seed ^ _ANCHOR_SALT)
    blocks = augment(plan, tokens, spec, prng)
    device = weights.embedding.device
    hosts = [Host(i) for i in range(plan.num_hosts)]
    # per host: its blocks in ascending order, and each block's first cache row
    row_of_block = {}
    for host in hosts:
        mine = plan.blocks_of(host.index)
        rows = sum(blocks[bi].own_len for bi in mine)
        host.pool = PagedKVPool(cfg.layers, cfg.heads, cfg.head_dim, max(rows, 1), page_size,
                                default_dtype(), device)
        r = 0
        for bi in mine:
            row_of_block[bi] = (host, r)
            r += blocks[bi].own_len
            host.pool.positions.extend(blocks[bi].own_positions)
    seg, pos = _block_rows(blocks)
    x = embed(weights, [t for bl in blocks for t in bl.token_ids])
    pos_t = torch.tensor(pos, dtype=torch.int64, device=device)
    dedup = _dedup_rows(plan, spec, blocks) if anchor_dedup else 0
    for li, lw in enumerate(weights.layers):
        q, k, v = project_qkv(x, lw, cfg, pos_t)
        att, _ = ops.phase1_fwd(q, k, v, seg, out_dtype=torch.float32, dedup_anchor_rows=dedup)
        for bi, bl in enumerate(blocks):
            lo = seg[bi] + bl.anchor_prefix_len
            host, r = row_of_block[bi]
            host.pool.write(li, k[lo:seg[bi + 1]], v[lo:seg[bi + 1]], r)
        x = finish_layer(x, att, lw)
    for host in hosts:
        if not plan.blocks_of(host.index):
            host.pool.layer_rows = [0] * cfg.layers
        host.channels = [KVCache(pool=host.pool, layer=li, head=h, host=host.index)
                         for li in range(cfg.layers) for h in range(cfg.heads)]
    return hosts


# ---------------------------------------------------------------------------- phase 2
def _partials_layer(hosts, qh: Host, layer: int, q: torch.Tensor, own_tail: int):
    """K2 on every host's pages for all heads: [(host, out [l, H, hd], lse [l, H])]."""
    parts = []
    l, H, hd = q.shape
    q4 = q.to(default_dtype()).view(1, l, H, hd).contiguous()
    for host in hosts:
        pool = host.pool
        n = pool.rows(layer)
        if n == 0:
            continue
        tail = own_tail if host is qh else 0
        o, s = ops.phase2_partial(q4.to(pool.dtype), pool.k[layer], pool.v[layer],
                                  pool.page_table.view(1, -1), pool.kv_len_tensor(layer), n,
                                  own_tail=tail)
        parts.append((host, o[0], s[0]))
    return parts


def _meter(ledger, qh, parts, l_q, d, heads):
    """Reference ledger order: per head, per non-query host (ss/sim.py:203-210)."""
    if ledger is None:
        return
    for _ in range(heads):
        for host, _, _ in parts:
            if host is not qh:
                ledger.append(2, host.index, qh.index, PARTIAL_OUT, l_q * d)
                ledger.append(2, host.index, qh.index, PARTIAL_LSE, l_q)


def _merge_parts(parts, l, H, hd):
    if not parts:
        raise ConfigError("every host cache is empty; nothing to attend to")
    if len(parts) == 1:
        return parts[0][1]
    outs = torch.stack([p[1].reshape(l * H, hd) for p in parts])
    lses = torch.stack([p[2].reshape(l * H) for p in parts])
    out, _ = ops.merge(outs, lses)
    return out.view(l, H, hd)


def _phase2_forward(hosts, weights: ModelWeights, token_ids, positions, own_tail: int,
                    ledger: CommLedger | None) -> torch.Tensor:
    """Append-then-attend on the query host, partials everywhere, ordered merge (ss/sim.py:254-281)."""
    cfg = weights.config
    qh = _query_host(hosts)
    if own_tail not in (0, len(token_ids)):
        raise ShapeError(f"own_tail must be 0 or the query length, got {own_tail}")
    x = embed(weights, token_ids)
    pos = list(positions)
    for li, lw in enumerate(weights.layers):
        q, k, v = project_qkv(x, lw, cfg, pos)
        qh.pool.append(li, k, v, pos)
        parts = _partials_layer(hosts, qh, li, q, own_tail)
        _meter(ledger, qh, parts, q.shape[0], cfg.head_dim, cfg.heads)
        att = _merge_parts(parts, q.shape[0], cfg.heads, cfg.head_dim)
        x = finish_layer(x, att, lw)
    return logits_from(weights, x)


def run_phase2_step(hosts: list[Host], q, own_tail: int = 0, ledger: CommLedger | None = None):
    """One distributed global-attention step per channel (ss/sim.py:216-237).

    q: one [l_q, d] query block (channel 0) or a sequence of per-channel blocks.
    Returns (merged output(s), ledger delta).
    """
    if not hosts:
        raise ConfigError("phase 2 requires at least one host")
    single = not isinstance(q, (list, tuple))
    qs = [q] if single else list(q)
    n_ch = min(len(h.channels) for h in hosts)
    if len(qs) > n_ch:
        raise ShapeError(f"{len(qs)} query channels but hosts expose {n_ch}")
    qh = _query_host(hosts)
    delta: list[LedgerEntry] = []
    outs = []
    for c, qc in enumerate(qs):
        qc = _as_device_2d(qc)
        if own_tail not in (0, qc.shape[0]):
            raise ShapeError(f"own_tail must be 0 or the query length, got {own_tail}")
        parts = []
        for host in hosts:
            cache = host.channels[c]
            if cache.rows == 0:
                continue
            pool = cache.pool
            # the channel's kv head as a one-head pool: K2 streams that head's rows only
            kh, vh, table = pool.head_view(cache.layer, cache.head)
            qq = qc.to(pool.dtype).reshape(1, qc.shape[0], 1, qc.shape[1]).contiguous()
            o, s = ops.phase2_partial(qq, kh, vh, table.view(1, -1),
                                      pool.kv_len_tensor(cache.layer), cache.rows,
                                      own_tail=own_tail if host is qh else 0)
            parts.append(PartialAttention(o[0, :, 0].to(qc.dtype), s[0, :, 0]))
            if host is not qh:
                for kind, count in ((PARTIAL_OUT, qc.shape[0] * qc.shape[1]),
                                    (PARTIAL_LSE, qc.shape[0])):
                    e = LedgerEntry(2, host.index, qh.index, kind, count)
                    delta.append(e)
                    if ledger is not None:
                        ledger.entries.append(e)
        if not parts:
            raise ConfigError("every host cache is empty; nothing to attend to")
        outs.append(merge_partials(parts).out)
    return (outs[0] if single else outs), delta


@dataclass
class DecodeSession:
    """State carried across autoregressive steps (ss/sim.py:240-251)."""

    hosts: list
    weights: ModelWeights
    ledger: CommLedger
    context_len: int
    query_len: int
    next_position: int
    last_logits: torch.Tensor
    generated: list = field(default_factory=list)
    _decoder: object = field(default=None, repr=False)  # decoding.DeviceDecoder, built lazily


def start_session(weights: ModelWeights, tokens, plan: BlockPlan, spec: AnchorSpec,
                  hosts: list[Host] | None = None, prng: Prng | None = None,
                  ledger: CommLedger | None = None, workers: int = 1):
    """Phase 1 on the context, then query encoding under phase 2 (ss/sim.py:284-324)."""
    L = plan.context_len
    tokens = list(tokens)
    if len(tokens) < L:
        raise ConfigError(f"{len(tokens)} tokens for a context of {L}")
    query = tokens[L:]
    if not query:
        raise ConfigError("query portion is empty; nothing to encode in phase 2")
    if hosts is None:
        hosts = run_phase1(tokens[:L], plan, spec, weights, prng=prng, workers=workers)
    ledger = ledger if ledger is not None else CommLedger()
    qh = _query_host(hosts)
    for h in hosts:
        if h is not qh:
            ledger.append(2, qh.index, h.index, QUERY_BROADCAST, len(query))
    logits = _phase2_forward(hosts, weights, query, range(L, L + len(query)), len(query), ledger)
    session = DecodeSession(hosts=hosts, weights=weights, ledger=ledger, context_len=L,
                            query_len=len(query), next_position=L + len(query),
                            last_logits=logits[-1])
    return logits, session


def forward_star(weights: ModelWeights, tokens, plan: BlockPlan, spec: AnchorSpec,
                 hosts: list[Host] | None = None, **kwargs) -> torch.Tensor:
    """Query-position logits under the two-phase path (ss/sim.py:327-337)."""
    logits, _ = start_session(weights, tokens, plan, spec, hosts=hosts, **kwargs)
    return logits


def _device_attend(hosts, qh: Host, max_rows: dict, theta: float, table=None):
    """Graph-safe phase-2 attention of one decode token (DeviceDecoder.attend_layer): append to
    the query host on the device, K2 on every non-empty host's pages with the device row
    counts, merge in ascending host order (ss/sim.py:254-281, :178-213)."""

    def attend(li, q, k, v, pos):
        qr = qh.pool.append_rope(li, q, k, v, pos, theta, table=table)
        H, hd = qr.shape[1], qr.shape[2]
        q4 = qr.view(1, 1, H, hd)
        parts = []
        for host in hosts:
            if max_rows[host.index] == 0:
                continue
            pool = host.pool
            o, s = ops.phase2_partial(q4, pool.k[li], pool.v[li], pool.page_table.view(1, -1),
                                      pool.kv_len_tensor(li), max_rows[host.index],
                                      workspace=pool.workspace)
            parts.append((host, o[0], s[0]))
        return _merge_parts(parts, 1, H, hd)

    return attend


def decode(session: DecodeSession, n_tokens: int, greedy: bool = True,
           graph: bool = True) -> list[int]:
    """Greedy decode, one phase-2 step per token (ss/sim.py:340-368).

    The step runs on the device (decoding.DeviceDecoder): argmax, embedding, append to the
    query host, K2 on every host, merge and the next logits, captured once in a CUDA graph
    and replayed per token; the ids come back in one read at the end.  The ledger gets the
    reference's rows (query broadcast, then per layer/head/non-query host the partials).
    """
    from .decoding import DeviceDecoder

    if not greedy:
        raise ConfigError("only greedy decoding is supported")
    if n_tokens <= 0:
        return []
    hosts = session.hosts
    qh = _query_host(hosts)
    cfg = session.weights.config
    dec = session._decoder
    if dec is None or dec.remaining() < n_tokens or dec.use_graph != graph:
        rows = qh.pool.rows(0)
        room = -(-max(n_tokens, 64) // 64) * 64
        qh.pool.reserve(rows + room, exact=True)
        max_rows = {h.index: h.pool.rows(0) for h in hosts}
        max_rows[qh.index] = rows + room
        table = ops.RopeTable(session.next_position, room, cfg.head_dim, cfg.rope_theta,
                              qh.pool.device)
        dec = DeviceDecoder(session.weights, session.last_logits, session.next_position,
                            _device_attend(hosts, qh, max_rows, cfg.rope_theta, table), room,
                            graph)
        session._decoder = dec
    new_tokens = dec.run(n_tokens)
    # host mirror of what the device step did
    p0 = session.next_position
    for li in range(cfg.layers):
        qh.pool.layer_rows[li] += n_tokens
    qh.pool.positions.extend(range(p0, p0 + n_tokens))
    nonempty = [(h, None, None) for h in hosts if h.pool.rows(0) > 0]
    for _ in new_tokens:
        for h in hosts:
            if h is not qh:
                session.ledger.append(2, qh.index, h.index, QUERY_BROADCAST, 1)
        for _li in range(cfg.layers):
            _meter(session.ledger, qh, nonempty, 1, cfg.head_dim, cfg.heads)
    session.generated.extend(new_tokens)
    session.next_position += n_tokens
    session.last_logits = dec.logits
    return new_tokens
