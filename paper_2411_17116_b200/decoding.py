"""Greedy decode with the whole per-token step on the device (ss/sim.py:340-368).

The reference's decode loop takes the argmax of the last logits on the host, embeds the
token, runs a phase-2 forward (append the token's K/V to the query host, partial attention
on every host, ordered merge) and repeats.  Here every piece of per-token state lives in
device memory — the logits, the token, its position, each pool's row counter
(`PagedKVPool.kv_len_dev`) and the exchange epochs — so one decode step is a fixed sequence
of launches.  The first step of a decoder runs eagerly (it sizes the workspaces and the
library's per-workspace state); the step is then captured in a CUDA graph and replayed once
per token.  The generated ids are read back with ONE device->host copy per `run` call.

Ties in the argmax go to the lowest id, as the reference's `int(np.argmax(...))`
(torch.argmax returns the first maximal index).

`attend_layer(li, q, k, v, pos)` is the protocol-specific part (single-process hosts in
sim.py, one rank per GPU in dist.py): given the new token's pre-RoPE q/k/v [1, H, hd] for
layer li and its position (device int64 [1]), it appends to the query host's pool on the
device and returns the merged attention output [1, H, hd].  It must be graph-safe: no host
reads of device values, no host-built tensors, fixed launch shapes.
"""

from __future__ import annotations

from typing import Callable

import torch

from . import ops
from .model import ModelWeights, finish_layer, logits_from, project_raw

AttendLayer = Callable[[int, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor], torch.Tensor]


class DeviceDecoder:
    """Device-resident greedy decode step for `capacity` tokens (graph-captured)."""

    def __init__(self, weights: ModelWeights, last_logits: torch.Tensor, next_position: int,
                 attend_layer: AttendLayer, capacity: int, graph: bool = True):
        dev = weights.embedding.device
        self.weights = weights
        self.device = dev
        self.logits = last_logits.detach().reshape(-1).float().clone()
        self.pos = torch.full((1,), int(next_position), dtype=torch.int64, device=dev)
        self.toks = torch.zeros(max(capacity, 1), dtype=torch.int64, device=dev)
        self.slot = torch.zeros(1, dtype=torch.int64, device=dev)
        self.attend_layer = attend_layer
        self.capacity = capacity
        self.used = 0
        self.use_graph = graph
        self.graph: torch.cuda.CUDAGraph | None = None
        self._stepped = False
        self.launches_per_step = None
        prime = getattr(attend_layer, "prime", None)
        if prime is not None:
            prime(self.pos)  # fused decode: cos/sin of the first position

    def _step(self) -> None:
        cfg = self.weights.config
        tok = torch.argmax(self.logits).view(1)
        self.toks.index_copy_(0, self.slot, tok)
        self.slot += 1
        x = self.weights.embedding.index_select(0, tok)
        for li, lw in enumerate(self.weights.layers):
            q, k, v = project_raw(x, lw, cfg)
            att = self.attend_layer(li, q, k, v, self.pos)
            x = finish_layer(x, att.view(1, cfg.heads, cfg.head_dim), lw)
        self.logits.copy_(logits_from(self.weights, x)[-1])
        finish = getattr(self.attend_layer, "finish", None)
        if finish is not None:
            finish(self.pos)  # fused decode: every layer's row counter and the position, 1 launch
        else:
            self.pos += 1

    def _capture(self) -> None:
        cur = torch.cuda.current_stream(self.device)
        side = torch.cuda.Stream(self.device)
        side.wait_stream(cur)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                self._step()
        cur.wait_stream(side)
        self.graph = g

    def remaining(self) -> int:
        return self.capacity - self.used

    def run(self, n: int) -> list[int]:
        """Decode n tokens; returns their ids (one device->host read)."""
        if n <= 0:
            return []
        if n > self.remaining():
            raise ValueError(f"decoder has room for {self.remaining()} more tokens, asked {n}")
        self.slot.zero_()
        for _ in range(n):
            if self.graph is not None:
                self.graph.replay()
            elif not self._stepped or not self.use_graph:
                self._step()  # eager: sizes workspaces before any capture
                self._stepped = True
            else:
                self._capture()
                self.graph.replay()
        self.used += n
        return [int(t) for t in self.toks[:n].tolist()]


def paged_attend(pool, *, appends: bool, max_rows: int, theta: float, heads: int,
                 exchange=None, group=None, rope_table=None, fused=None) -> AttendLayer:
    """Graph-safe phase-2 attention of one decode token against this rank's paged cache
    `pool` (the DeviceDecoder `attend_layer` of one rank; also the bench's 32-layer step).

    appends: this rank is the query host — the token's rotated k and raw v are appended at
    the device row counter first (append-then-attend, ss/sim.py:275-277).  max_rows: the
    fixed K2 key bound for every replay (rows now + the token budget on the query host).
    exchange: a dist.PeerExchange — one K2 kernel computes the partial, stores it into every
    rank's box and merges every rank's partial (C1 fused); None with a process group: K2 +
    one all-gather of the packed partial + K3; None without a group: K2 alone (one host).
    A rank with no rows pushes an empty partial (lse = -inf) so the merge stays collective.
    rope_table: ops.RopeTable of the decode positions (the append then reads cos/sin instead
    of forming fp64 angles per token; bit-identical), or an ops.DecodeRope (its table plus the
    cos/sin at the current position, refreshed by .finish: the fused K2 then reads them with
    no dependent position load).
    fused: one launch per layer (ops.phase2_decode: RoPE + append inside K2; the returned
    attend then has .finish(pos), which the decoder calls once per token to advance every
    layer's row counter and the position).  Default: whenever the pool allows it (bf16,
    page_size % 64 == 0, head_dim 64/128) and this rank holds rows.
    Returns the merged attention [1, H, hd] (fp32)."""
    H, hd = heads, pool.head_dim
    hkv = pool.hkv
    mine = max_rows > 0
    # fused decode (star_phase2_decode): RoPE and the append inside K2, the row counters
    # advanced once per token by attend.finish — one launch per layer instead of two
    fused = (fused if fused is not None else
             (pool.dtype == torch.bfloat16 and hd in (64, 128) and pool.page_size % 64 == 0
              and H // hkv <= 16 and mine))

    def attend_fused(li, q, k, v, pos):
        qb = q.reshape(1, H, hd).to(pool.dtype)
        kb = k.reshape(1, hkv, hd).to(pool.dtype) if appends else None
        vb = v.reshape(1, hkv, hd).to(pool.dtype) if appends else None
        kv = (pool.k[li], pool.v[li], pool.page_table.view(1, -1), pool.kv_len_tensor(li))
        if exchange is not None:
            att, _ = exchange.decode_exchange(qb, kb, vb, pos, *kv, max_rows, theta, rope_table,
                                              appends, workspace=pool.workspace)
            return att.view(1, H, hd)
        if group is None:
            att, _ = ops.phase2_decode(qb, kb, vb, pos, *kv, max_rows, theta, rope_table, appends,
                                       workspace=pool.workspace)
            return att.view(1, H, hd)
        from .dist import gather_merge

        packed, o, s = ops.packed_partial(H, hd, q.device)
        ops.phase2_decode(qb, kb, vb, pos, *kv, max_rows, theta, rope_table, appends,
                          out=o.view(1, 1, H, hd), lse=s.view(1, 1, H), workspace=pool.workspace)
        att, _ = gather_merge(o, s, group=group, packed=packed)
        return att.view(1, H, hd)

    rope = rope_table if isinstance(rope_table, ops.DecodeRope) else None
    flat_table = rope_table.table if rope is not None else rope_table

    def finish(pos):
        ops.decode_advance(pool.kv_len_dev if appends else pool.kv_len_dev[:0], pos, rope=rope)

    def prime(pos):
        if rope is not None:
            rope.prime(pos)

    def attend(li, q, k, v, pos):
        if appends:
            qr = pool.append_rope(li, q, k, v, pos, theta, table=flat_table)
        else:
            qr = ops.rope(q.to(pool.dtype).contiguous(), pos, theta)
        qb = qr.view(1, 1, H, hd)
        kv = (pool.k[li], pool.v[li], pool.page_table.view(1, -1), pool.kv_len_tensor(li))
        if exchange is not None:
            if mine:
                att, _ = exchange.exchange(qb, *kv, max_rows, workspace=pool.workspace)
                return att.view(1, H, hd)
            exchange.push(torch.zeros(H, hd, device=q.device),
                          torch.full((H,), float("-inf"), device=q.device), 1, 1, H, hkv)
            att, _ = exchange.merge(1, 1, H, hkv)
            return att.view(1, H, hd)
        if group is None:
            att, _ = ops.phase2_partial(qb, *kv, max_rows, workspace=pool.workspace)
            return att.view(1, H, hd)
        from .dist import gather_merge

        packed, o, s = ops.packed_partial(H, hd, q.device)
        if mine:
            ops.phase2_partial(qb, *kv, max_rows, out=o.view(1, 1, H, hd), lse=s.view(1, 1, H),
                               workspace=pool.workspace)
        else:
            o.zero_()
            s.fill_(float("-inf"))
        att, _ = gather_merge(o, s, group=group, packed=packed)
        return att.view(1, H, hd)

    if fused:
        attend_fused.finish = finish
        attend_fused.prime = prime
        return attend_fused
    return attend
