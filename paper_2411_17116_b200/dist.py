"""Star attention across GPU ranks: one host per rank (torch.distributed + NCCL).

Phase 1 is rank-local: rank r encodes exactly the blocks partition() assigns it
(ss/blocking.py:68) into its own paged pool; no communication.  Phase 2 per
layer: every rank runs K2 over its pages and every rank ends up with every
rank's fp32 (out, lse) partial (16.5 KB per rank at B = l_q = 1 for Llama-8B
shapes), folded in ascending rank order — the reference's fixed host order
(ss/sim.py:189-213).  Two transports: the fused one (PeerExchange), where K2's
epilogue stores the partial into every rank's box over NVLink peer memory and
K3x merges once all flags are up; and one all-gather of the packed partials +
K3 over the process group's backend (NCCL or gloo).  All-gather rather than
gather-to-query-host closes the reference's unmetered return path: every rank
gets the merged attention and can compute layer l+1's queries.
The ledger records the reference's logical transfers on the query rank.

The collective / merge / ledger helpers are backend-agnostic (any
torch.distributed backend, an injectable merge function) so the host logic is
tested with gloo on CPU (tests/test_dist_cpu.py).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Callable

import torch
import torch.distributed as dist

from .blocking import AnchorSpec, BlockPlan, PagedKVPool, augment
from .errors import ConfigError
from .numerics import Prng, default_dtype

_ANCHOR_SALT = 0xA17C4B10C4ED5EED


def init_from_env(backend: str = "nccl") -> tuple[int, int]:
    """Initialise the default process group from torchrun's env; returns (rank, world)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            local = int(os.environ.get("LOCAL_RANK", "0"))
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world


@dataclass(frozen=True)
class RankShard:
    """What one rank owns in phase 1: its blocks (ascending), their own rows and positions."""

    rank: int
    blocks: tuple[int, ...]
    seg_start: tuple[int, ...]       # augmented-row offsets of the rank's blocks (segments)
    own_lo: tuple[int, ...]          # first own row of each block inside the segments
    cache_row0: tuple[int, ...]      # first cache row of each block in the rank's pool
    positions: tuple[int, ...]       # position ids of every augmented row, block order
    cache_positions: tuple[int, ...]  # position ids of the cached (own) rows

    @property
    def rows(self) -> int:
        return self.seg_start[-1]

    @property
    def cache_rows(self) -> int:
        return len(self.cache_positions)


def rank_shard(plan: BlockPlan, blocks_aug, rank: int) -> RankShard:
    """Host logic of the phase-1 sharding (ss/sim.py:148-174, one host per rank)."""
    mine = plan.blocks_of(rank)
    seg, lo, c0, pos, cpos = [0], [], [], [], []
    for bi in mine:
        bl = blocks_aug[bi]
        lo.append(seg[-1] + bl.anchor_prefix_len)
        c0.append(len(cpos))
        seg.append(seg[-1] + len(bl.token_ids))
        pos.extend(bl.position_ids)
        cpos.extend(bl.own_positions)
    return RankShard(rank, tuple(mine), tuple(seg), tuple(lo), tuple(c0), tuple(pos), tuple(cpos))


def gather_packed(packed: torch.Tensor, group=None) -> torch.Tensor:
    """ONE all-gather of every rank's packed partial [rows*d out | rows lse] -> [world, rows*(d+1)]."""
    world = dist.get_world_size(group)
    if packed.is_cuda and dist.get_backend(group) != "nccl":
        # host-staged collective (gloo: the multi-rank test backend): an explicit device->host
        # read and host->device write, so the result never depends on a CPU backend's handling
        # of CUDA-stream ordering
        host = packed.contiguous().view(-1).cpu()
        parts = torch.empty(world * host.numel(), dtype=host.dtype)
        dist.all_gather_into_tensor(parts, host, group=group)
        return parts.to(packed.device).view(world, packed.numel())
    parts = torch.empty(world * packed.numel(), dtype=packed.dtype, device=packed.device)
    dist.all_gather_into_tensor(parts, packed.contiguous().view(-1), group=group)
    return parts.view(world, packed.numel())


def gather_partials(out: torch.Tensor, lse: torch.Tensor, group=None):
    """All-gather one partial per rank: out [rows, d] fp32, lse [rows] -> [world, rows, d], [world, rows].

    Both travel in one packed collective (the wire format of SURVEY §8e: l_q*Hq*(d+1) fp32
    per rank)."""
    rows, d = out.shape[0], out[0].numel()
    packed = torch.cat([out.reshape(-1), lse.reshape(-1)])
    parts = gather_packed(packed, group)
    world = parts.shape[0]
    return (parts[:, :rows * d].reshape((world,) + tuple(out.shape)),
            parts[:, rows * d:].reshape(world, rows))


def gather_merge(out: torch.Tensor, lse: torch.Tensor, merge_fn: Callable | None = None,
                 group=None, packed: torch.Tensor | None = None):
    """All-gather the ranks' partials and fold them in ascending rank order (ranks whose
    cache is empty contribute lse = -inf and are skipped, ss/sim.py:193-194).

    `packed`, when given, is the buffer `out`/`lse` are views of (ops.packed_partial): the
    collective then sends it as is and K3 reads the gathered parts in place."""
    if merge_fn is None and out.is_cuda:
        from . import ops

        rows, d = out.shape[0], out[0].numel()
        if packed is None:
            packed = torch.cat([out.reshape(-1), lse.reshape(-1)])
        return ops.merge_packed(gather_packed(packed, group), rows, d)
    outs, lses = gather_partials(out, lse, group)
    if merge_fn is None:
        from . import ops

        merge_fn = ops.merge
    return merge_fn(outs, lses)


class PeerExchange:
    """One rank's end of the fused phase-2 exchange (C1 over NVLink peer memory).

    Replaces the NCCL all-gather + K3 of gather_merge: K2's epilogue stores the rank's final
    partial straight into slot `rank` of every rank's box and raises a flag; K3x waits for
    all ranks' flags in the local box and merges in ascending rank order (the reference's
    fixed host order, ss/sim.py:189-213).  Layout / protocol: csrc/exchange.cuh.

    `boxes` are device addresses, one per rank (boxes[rank] is this rank's own box, the
    others are CUDA-IPC mappings).  Every rank runs the same sequence of exchanges (push,
    then merge); the exchanges are numbered by a counter in each box that K3x advances, so
    they stay in step without host bookkeeping and a captured decode graph replays.
    """

    def __init__(self, rank: int, boxes: list[int], cap_rows: int, cap_groups: int, d: int,
                 own_box: torch.Tensor, opened: list[tuple[int, int]] | None = None):
        self.rank, self.boxes = rank, list(boxes)
        self.world = len(boxes)
        self.cap_rows, self.cap_groups, self.d = cap_rows, cap_groups, d
        self.own_box = own_box
        self._opened = opened or []

    def fits(self, batch: int, lq: int, hq: int, hkv: int, d: int) -> bool:
        return batch * lq * hq <= self.cap_rows and batch * hkv <= self.cap_groups and d == self.d

    def push_partial(self, q, k_pages, v_pages, page_table, kv_len, max_kv_len,
                     own_tail: int = 0, n_splits: int = 0, workspace=None) -> None:
        from . import ops

        ops.phase2_partial_push(q, k_pages, v_pages, page_table, kv_len, max_kv_len, self.boxes,
                                self.cap_rows, self.cap_groups, self.rank, own_tail, n_splits,
                                workspace)

    def exchange(self, q, k_pages, v_pages, page_table, kv_len, max_kv_len, own_tail: int = 0,
                 n_splits: int = 0, workspace=None):
        """Partial over the local cache + push + merge of every rank's partial (one kernel
        when possible).  Returns fp32 (out [B, lq, hq, d], lse [B, lq, hq])."""
        from . import ops

        return ops.phase2_exchange(q, k_pages, v_pages, page_table, kv_len, max_kv_len,
                                   self.boxes, self.cap_rows, self.cap_groups, self.rank,
                                   own_tail, n_splits, workspace)

    def decode_exchange(self, q, k, v, positions, k_pages, v_pages, page_table, kv_len,
                        max_kv_len, theta, table=None, append=True, n_splits: int = 0,
                        workspace=None):
        """Fused decode step (RoPE + append inside K2) + push + merge of every rank's partial
        (ops.phase2_decode_exchange).  Returns fp32 (out [B, 1, hq, d], lse [B, 1, hq])."""
        from . import ops

        return ops.phase2_decode_exchange(q, k, v, positions, k_pages, v_pages, page_table,
                                          kv_len, max_kv_len, self.boxes, self.cap_rows,
                                          self.cap_groups, self.rank, theta, table, append,
                                          n_splits, workspace)

    def push(self, out, lse, batch, lq, hq, hkv) -> None:
        from . import ops

        ops.exchange_push(out, lse, batch, lq, hq, hkv, self.boxes, self.cap_rows,
                          self.cap_groups, self.rank)

    def merge(self, batch, lq, hq, hkv, out_dtype=torch.float32):
        from . import ops

        return ops.exchange_merge(self.boxes[self.rank], self.world, self.cap_rows,
                                  self.cap_groups, batch, lq, hq, hkv, self.d,
                                  self.own_box.device, out_dtype)

    def close(self) -> None:
        from . import ops

        for ptr, off in self._opened:
            ops.ipc_close_handle(ptr, off)
        self._opened = []


def _alloc_box(world, cap_rows, cap_groups, d, device) -> torch.Tensor:
    from . import ops

    n = ops.exchange_box_bytes(world, cap_rows, cap_groups, d)
    return torch.zeros(n, dtype=torch.uint8, device=device)


class PeerExchangeUnavailable(RuntimeError):
    """Raised on EVERY rank when any rank cannot map the exchange boxes (no CUDA IPC, e.g.
    virtual-memory allocations or ranks without peer access); callers fall back to the
    all-gather transport."""


def open_peer_exchange(cap_rows: int, cap_groups: int, d: int, device, group=None) -> PeerExchange:
    """Collective: allocate this rank's box, swap CUDA-IPC handles with every rank (one
    all_gather_object over `group`, any backend) and map the peers' boxes.  Every rank gets
    the same outcome: a PeerExchange, or PeerExchangeUnavailable."""
    from . import ops

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    box = _alloc_box(world, cap_rows, cap_groups, d, device)
    torch.cuda.synchronize(device)  # the zeroed box is visible before any peer can write it
    try:
        handle, off = ops.ipc_get_handle(box)
        mine = (True, handle, off, "")
    except Exception as exc:  # noqa: BLE001 - reported collectively below
        mine = (False, b"", 0, f"rank {rank}: {exc}")
    allh = [None] * world
    dist.all_gather_object(allh, mine, group=group)
    bad = [m[3] for m in allh if not m[0]]
    if bad:
        raise PeerExchangeUnavailable("; ".join(bad))
    boxes, opened, err = [], [], ""
    for r, (_, h, o, _) in enumerate(allh):
        if r == rank:
            boxes.append(box.data_ptr())
            continue
        try:
            ptr = ops.ipc_open_handle(h, o)
        except Exception as exc:  # noqa: BLE001
            err = f"rank {rank} mapping rank {r}: {exc}"
            break
        boxes.append(ptr)
        opened.append((ptr, o))
    status = [None] * world
    dist.all_gather_object(status, err, group=group)
    if any(status):
        for ptr, o in opened:
            ops.ipc_close_handle(ptr, o)
        raise PeerExchangeUnavailable("; ".join(x for x in status if x))
    dist.barrier(group=group)  # every box mapped everywhere before the first exchange
    return PeerExchange(rank, boxes, cap_rows, cap_groups, d, box, opened)


def local_peer_exchanges(world: int, cap_rows: int, cap_groups: int, d: int,
                         device) -> list[PeerExchange]:
    """`world` ranks' boxes in ONE process (tests, and the single-GPU bench of the exchange
    path): same kernels and layout, plain device pointers instead of IPC mappings."""
    boxes = [_alloc_box(world, cap_rows, cap_groups, d, device) for _ in range(world)]
    ptrs = [b.data_ptr() for b in boxes]
    return [PeerExchange(r, ptrs, cap_rows, cap_groups, d, boxes[r]) for r in range(world)]


def phase2_ledger_rows(q_rank: int, nonempty_ranks, layers: int, heads: int, l_q: int, d: int):
    """Ledger rows one phase-2 forward emits, in the reference's order (ss/sim.py:203-210)."""
    rows = []
    for _ in range(layers):
        for _ in range(heads):
            for r in nonempty_ranks:
                if r != q_rank:
                    rows.append((2, r, q_rank, "partial_out", l_q * d))
                    rows.append((2, r, q_rank, "partial_lse", l_q))
    return rows


@dataclass
class DistSession:
    """Per-rank state of a distributed two-phase session."""

    weights: object
    plan: BlockPlan
    shard: RankShard
    pool: PagedKVPool
    q_rank: int
    ledger: list = field(default_factory=list)
    next_position: int = 0
    last_logits: torch.Tensor | None = None
    generated: list = field(default_factory=list)
    exchange: PeerExchange | None = None  # fused C1 transport; None = all-gather + K3
    # ranks holding cache rows in phase 2, ascending: the plan's block owners plus the query
    # rank (fixed once phase 1 is done; no per-token collective needed)
    nonempty: list = field(default_factory=list)
    _decoder: object = field(default=None, repr=False)  # decoding.DeviceDecoder


def run_phase1_dist(tokens, plan: BlockPlan, spec: AnchorSpec, weights, prng: Prng | None = None,
                    group=None, page_size: int = 128) -> tuple[RankShard, PagedKVPool]:
    """Phase 1 on this rank's blocks only (no communication)."""
    from . import ops
    from .model import embed, finish_layer, project_qkv

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if world != plan.num_hosts:
        raise ConfigError(f"plan has {plan.num_hosts} hosts but the group has {world} ranks")
    cfg = weights.config
    prng = prng or Prng(cfg.seed ^ _ANCHOR_SALT)
    blocks = augment(plan, tokens, spec, prng)  # identical on every rank (deterministic)
    shard = rank_shard(plan, blocks, rank)
    dev = weights.embedding.device
    pool = PagedKVPool(cfg.layers, cfg.heads, cfg.head_dim, max(shard.cache_rows, 1), page_size,
                       default_dtype(), dev)
    pool.positions.extend(shard.cache_positions)
    if shard.blocks:
        x = embed(weights, [t for bi in shard.blocks for t in blocks[bi].token_ids])
        pos = torch.tensor(shard.positions, dtype=torch.int64, device=dev)
        for li, lw in enumerate(weights.layers):
            q, k, v = project_qkv(x, lw, cfg, pos)
            att, _ = ops.phase1_fwd(q, k, v, list(shard.seg_start), out_dtype=torch.float32)
            for j, bi in enumerate(shard.blocks):
                lo, hi = shard.own_lo[j], shard.seg_start[j + 1]
                pool.write(li, k[lo:hi], v[lo:hi], shard.cache_row0[j])
            x = finish_layer(x, att, lw)
    return shard, pool


def _phase2_forward_dist(sess: DistSession, token_ids, positions, own_tail: int, group=None):
    from . import ops
    from .model import embed, finish_layer, logits_from, project_qkv

    cfg = sess.weights.config
    rank = dist.get_rank(group)
    x = embed(sess.weights, token_ids)
    pos = list(positions)
    H, hd = cfg.heads, cfg.head_dim
    for li, lw in enumerate(sess.weights.layers):
        q, k, v = project_qkv(x, lw, cfg, pos)
        if rank == sess.q_rank:
            sess.pool.append(li, k, v, pos)
        l = q.shape[0]
        n = sess.pool.rows(li)
        qb = q.view(1, l, H, hd).to(sess.pool.dtype).contiguous()
        tail = own_tail if rank == sess.q_rank else 0
        ex = sess.exchange
        if ex is not None:
            # fused C1: K2 stores its partial into every rank's box, K3x merges (no NCCL)
            hkv = sess.pool.k[li].shape[1]
            if n:
                att, _ = ex.exchange(qb, sess.pool.k[li], sess.pool.v[li],
                                     sess.pool.page_table.view(1, -1),
                                     sess.pool.kv_len_tensor(li), n, own_tail=tail,
                                     workspace=sess.pool.workspace)
                att = att.view(l * H, hd)
            else:
                ex.push(torch.zeros(l * H, hd, device=q.device),
                        torch.full((l * H,), float("-inf"), device=q.device), 1, l, H, hkv)
                att, _ = ex.merge(1, l, H, hkv)
        else:
            packed, o, s = ops.packed_partial(l * H, hd, q.device)
            if n:
                ops.phase2_partial(qb, sess.pool.k[li], sess.pool.v[li],
                                   sess.pool.page_table.view(1, -1), sess.pool.kv_len_tensor(li),
                                   n, own_tail=tail, out=o.view(1, l, H, hd), lse=s.view(1, l, H),
                                   workspace=sess.pool.workspace)
            else:
                o.zero_()
                s.fill_(float("-inf"))
            att, _ = gather_merge(o, s, group=group, packed=packed)
        x = finish_layer(x, att.view(l, H, hd), lw)
    if rank == sess.q_rank:
        sess.ledger.extend(phase2_ledger_rows(sess.q_rank, sess.nonempty, cfg.layers, H, len(pos),
                                              hd))
    return logits_from(sess.weights, x)


def start_session_dist(weights, tokens, plan: BlockPlan, spec: AnchorSpec, prng=None,
                       q_rank: int | None = None, group=None, transport: str = "auto"):
    """Distributed start_session (ss/sim.py:284-324): phase 1 per rank, then the query.

    transport: "peer" = fused C1 over CUDA-IPC peer memory (PeerExchange; all ranks on one
    node), "collective" = one all-gather of the packed partials + K3 over the process group's
    backend, "auto" = peer when the group runs NCCL (one GPU per rank), else collective."""
    if transport not in ("auto", "peer", "collective"):
        raise ConfigError(f"unknown phase-2 transport {transport!r}")
    auto = transport == "auto"
    if auto:
        transport = "peer" if dist.get_backend(group) == "nccl" else "collective"
    world = dist.get_world_size(group)
    L = plan.context_len
    tokens = list(tokens)
    query = tokens[L:]
    if not query:
        raise ConfigError("query portion is empty; nothing to encode in phase 2")
    shard, pool = run_phase1_dist(tokens[:L], plan, spec, weights, prng, group)
    q_rank = world - 1 if q_rank is None else q_rank
    sess = DistSession(weights, plan, shard, pool, q_rank)
    sess.nonempty = [r for r in range(world) if plan.blocks_of(r) or r == q_rank]
    if transport == "peer":
        cfg = weights.config
        # capacity: the query encode's l_q rows x heads (decode steps use a prefix of it)
        try:
            sess.exchange = open_peer_exchange(len(query) * cfg.heads, pool.k[0].shape[1],
                                               cfg.head_dim, weights.embedding.device, group)
        except PeerExchangeUnavailable:
            if not auto:
                raise
            sess.exchange = None  # every rank falls back to the all-gather transport
    if dist.get_rank(group) == q_rank:
        sess.ledger += [(2, q_rank, r, "query_broadcast", len(query)) for r in range(world)
                        if r != q_rank]
    logits = _phase2_forward_dist(sess, query, range(L, L + len(query)), len(query), group)
    sess.next_position = L + len(query)
    sess.last_logits = logits[-1]
    return logits, sess


def decode_dist(sess: DistSession, n_tokens: int, group=None, graph: bool | None = None) -> list[int]:
    """Distributed greedy decode (ss/sim.py:340-368); every rank derives the same token.

    The per-token step runs on the device (decoding.DeviceDecoder) and is graph-captured
    when the transport allows it (the peer exchange, or NCCL collectives; a gloo group runs
    the same device step eagerly).  No collective or host sync per token: the ids are read
    back once per call."""
    from . import ops
    from .decoding import DeviceDecoder, paged_attend

    if n_tokens <= 0:
        return []
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    cfg = sess.weights.config
    if graph is None:
        graph = sess.exchange is not None or dist.get_backend(group) == "nccl"
    dec = sess._decoder
    if dec is None or dec.remaining() < n_tokens or dec.use_graph != graph:
        rows = sess.pool.rows(0)
        room = -(-max(n_tokens, 64) // 64) * 64 if rank == sess.q_rank else 0
        if room:
            sess.pool.reserve(rows + room, exact=True)
        # every rank sizes its decoder for the same token budget
        budget = -(-max(n_tokens, 64) // 64) * 64
        # (paged_attend's group=None means one host: pass the process group explicitly)
        # cos/sin of the token budget's positions on every rank: the query rank's append and
        # every rank's in-kernel q rotation (fused decode) read it
        table = ops.DecodeRope(sess.next_position, budget, cfg.head_dim, cfg.rope_theta, 1,
                               sess.pool.device)
        attend = paged_attend(sess.pool, appends=rank == sess.q_rank,
                              max_rows=rows + room if rank in sess.nonempty else 0,
                              theta=cfg.rope_theta, heads=cfg.heads, exchange=sess.exchange,
                              group=group if group is not None else dist.group.WORLD,
                              rope_table=table)
        dec = DeviceDecoder(sess.weights, sess.last_logits, sess.next_position, attend, budget,
                            graph)
        sess._decoder = dec
    out = dec.run(n_tokens)
    p0 = sess.next_position
    if rank == sess.q_rank:
        for li in range(cfg.layers):
            sess.pool.layer_rows[li] += n_tokens
        sess.pool.positions.extend(range(p0, p0 + n_tokens))
        for _ in out:
            sess.ledger += [(2, sess.q_rank, r, "query_broadcast", 1) for r in range(world)
                            if r != sess.q_rank]
            sess.ledger.extend(phase2_ledger_rows(sess.q_rank, sess.nonempty, cfg.layers,
                                                  cfg.heads, 1, cfg.head_dim))
    sess.generated.extend(out)
    sess.next_position += n_tokens
    sess.last_logits = dec.logits
    return out
