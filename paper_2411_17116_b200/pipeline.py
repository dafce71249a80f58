"""Host-buffer entry point of the phase-1 encode, pipelined per block.

The reference's phase 1 takes host (numpy) data and returns host data
(ss/sim.py:126-175).  Called with pinned host tensors, this module overlaps,
per anchor-augmented block (segment): host->device copy of block i+1, the fused
prologue (RoPE + own-row KV page write) and K1 of block i, device->host copy of the output of block i-1 —
on CUDA streams ordered by events: one for the H2D copies, one for the D2H copies and two
for compute, taken by alternate blocks — blocks are independent (a block's K1 reads only its
own rows), so the next block's prologue and K1 fill the SMs the current block's last CTAs
leave idle instead of waiting for its launch to drain.  The copies then hide behind the
tensor-core work instead of adding to it.

Two host input layouts:
  * augmented (`encode_layer_host`): q/k/v rows exactly as the augmented blocks are
    laid out, anchor rows repeated per block (ss/blocking.py:206-236);
  * context (`encode_layer_host_context`): each distinct context row once.  With
    first-block anchors (content and positions, the reference default) a block's anchor
    rows are block 0's rows bit for bit at every layer (same tokens, positions and causal
    prefix), so they cross PCIe once and are replicated on the device; every augmented row
    is still encoded and returned.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Sequence

import torch

from . import ops
from .errors import ShapeError


@dataclass
class LayerEncodePlan:
    """Device buffers and streams for repeated host-buffer encodes of one layer shape."""

    seg: list
    own: list            # own rows per segment (the tail of each segment)
    cache_row0: list     # first cache row of each segment's own rows
    q: torch.Tensor      # device staging, [rows, hq, d]
    k: torch.Tensor
    v: torch.Tensor
    q_rot: torch.Tensor
    k_rot: torch.Tensor
    out: torch.Tensor
    cache_rows: torch.Tensor  # logical cache row per augmented row, -1 for anchor rows
    streams: tuple = field(default_factory=tuple)
    # context layout: per segment, (dev_row, ctx_row, n) host->device ranges and
    # (dst_row, src_row, n) device->device ranges (rows already on the device)
    ctx_rows: int = 0
    h2d: list = field(default_factory=list)
    d2d: list = field(default_factory=list)
    # cross-call ordering of back-to-back encodes (wait=False): per segment, the previous
    # call's last compute (it read the staging rows the next H2D overwrites) and last D2H
    # (it read the output rows the next K1 overwrites); `done` = the last call finished
    comp_done: list = field(default_factory=list)
    d2h_done: list = field(default_factory=list)
    done: object = None

    def synchronize(self) -> None:
        """Block the host until the last encode (including its D2H) has finished."""
        if self.done is not None:
            self.done.synchronize()

    @classmethod
    def create(cls, seg: Sequence[int], own: Sequence[int], hq: int, hkv: int, d: int,
               device, dtype=torch.bfloat16) -> "LayerEncodePlan":
        rows = seg[-1]
        if len(own) != len(seg) - 1:
            raise ShapeError("one own-row count per segment")
        c0, acc = [], 0
        for o in own:
            c0.append(acc)
            acc += o
        mk = lambda h: torch.empty((rows, h, d), dtype=dtype, device=device)  # noqa: E731
        q, k, v = mk(hq), mk(hkv), mk(hkv)
        cr = torch.full((rows,), -1, dtype=torch.int64)
        for i, o in enumerate(own):
            cr[seg[i + 1] - o:seg[i + 1]] = torch.arange(c0[i], c0[i] + o)
        # H2D, compute (even blocks), D2H, compute (odd blocks)
        streams = tuple(torch.cuda.Stream(device) for _ in range(4))
        return cls(list(seg), list(own), c0, q, k, v, torch.empty_like(q), torch.empty_like(k),
                   torch.empty_like(q), cr.to(device), streams)

    def set_context_layout(self, positions) -> int:
        """Derive the context-layout copy plan from the augmented rows' context positions
        (first-block anchors: a row's position is its context row).  Returns the number of
        distinct context rows, i.e. the rows of the host buffers to pass."""
        import numpy as np

        pos = np.asarray(positions, dtype=np.int64)
        if pos.shape[0] != self.seg[-1]:
            raise ShapeError("one position per augmented row")
        uniq = np.unique(pos)
        ctx = np.searchsorted(uniq, pos)
        placed = []  # (ctx_start, dev_start, n) ranges already on the device
        self.h2d, self.d2d = [], []
        for i in range(len(self.seg) - 1):
            a_i = (self.seg[i + 1] - self.seg[i]) - self.own[i]
            parts = [(self.seg[i], a_i), (self.seg[i] + a_i, self.own[i])]
            h, dd = [], []
            for r0, n in parts:
                if n == 0:
                    continue
                c0 = int(ctx[r0])
                if not np.array_equal(ctx[r0:r0 + n], np.arange(c0, c0 + n)):
                    raise ShapeError("context layout needs contiguous context rows per part")
                src = next((d0 + (c0 - s0) for s0, d0, m in placed if s0 <= c0 and c0 + n <= s0 + m),
                           None)
                if src is None:
                    h.append((r0, c0, n))
                    placed.append((c0, r0, n))
                else:
                    dd.append((r0, src, n))
            self.h2d.append(h)
            self.d2d.append(dd)
        self.ctx_rows = int(uniq.shape[0])
        return self.ctx_rows


# query-row cut fractions of the first and last segments (fill and drain of the pipeline);
# STAR_E2E_CUTS="0.125,0.25,0.5/0.5,0.75,0.875" overrides them (measurement knob)
FIRST_CUTS = (0.5,)
LAST_CUTS = (0.5, 0.75)


def _cut_fracs():
    import os

    env = os.environ.get("STAR_E2E_CUTS")
    if not env:
        return FIRST_CUTS, LAST_CUTS
    f, l = env.split("/")
    return (tuple(float(x) for x in f.split(",") if x), tuple(float(x) for x in l.split(",") if x))


def _cuts(m: int, first: bool, last: bool) -> list:
    """Query-row cut points of one segment: the first segment is encoded in causal parts (the
    H2D of a later part overlaps the K1 of an earlier one), the last in parts whose D2H
    overlaps the K1 of the rest; interior segments whole.  Cuts land on 128-row q tiles."""
    fc, lc = _cut_fracs()
    pts = {0, m}
    if first:
        pts.update(int(m * f) for f in fc)
    if last:
        pts.update(int(m * f) for f in lc)
    return sorted({min(m, (c // 128) * 128) if c not in (0, m) else c for c in pts})


def _clip(ranges, lo: int, hi: int):
    """(dst_row, src_row, n) ranges restricted to destination rows [lo, hi)."""
    out = []
    for r0, src, n in ranges:
        a, b = max(r0, lo), min(r0 + n, hi)
        if a < b:
            out.append((a, src + (a - r0), b - a))
    return out


def _encode(plan: LayerEncodePlan, copy_in, positions, k_pages, v_pages, page_table, out_host,
            theta, wait: bool = True):
    """Per segment and query-row part: H2D (copy_in) | RoPE + KV write + K1 range | D2H.

    wait=False returns without making the current stream wait for the pipeline, so the next
    call's H2D (fill) overlaps this call's last D2H (drain) and compute; cross-call hazards on
    the staging and output rows are ordered per segment by events (plan.comp_done / d2h_done).
    The caller then waits on plan.done (an event) or calls plan.synchronize()."""
    s_in, s_comp0, s_out, s_comp1 = plan.streams
    comps = (s_comp0, s_comp1) if os.environ.get("STAR_E2E_COMP1", "0") != "1" else (s_comp0,)
    cur = torch.cuda.current_stream(plan.q.device)
    start = torch.cuda.Event()
    start.record(cur)
    for st in (s_in, s_out) + comps:
        st.wait_event(start)
    n = len(plan.seg) - 1
    if len(plan.comp_done) != n:
        plan.comp_done, plan.d2h_done = [None] * n, [None] * n
    for i in range(n):
        a, b = plan.seg[i], plan.seg[i + 1]
        s_comp = comps[i % len(comps)]
        cuts = _cuts(b - a, i == 0, i == n - 1)
        for k_part, (p0, p1) in enumerate(zip(cuts[:-1], cuts[1:])):
            with torch.cuda.stream(s_in):
                if k_part == 0 and plan.comp_done[i] is not None:
                    s_in.wait_event(plan.comp_done[i])
                copy_in(i, a + p0, a + p1)
            ev_in = torch.cuda.Event()
            ev_in.record(s_in)
            with torch.cuda.stream(s_comp):
                s_comp.wait_event(ev_in)
                if k_part == 0 and plan.d2h_done[i] is not None:
                    s_comp.wait_event(plan.d2h_done[i])
                r0, r1 = a + p0, a + p1
                ops.rope_qkv(plan.q[r0:r1], plan.k[r0:r1], plan.v[r0:r1], positions[r0:r1], theta,
                             q_out=plan.q_rot[r0:r1], k_out=plan.k_rot[r0:r1],
                             cache_rows=plan.cache_rows[r0:r1], k_pages=k_pages,
                             v_pages=v_pages, page_table=page_table)
                # causal: query rows [p0, p1) need keys [0, p1) only — already rotated
                ops.phase1_fwd_range(plan.q_rot[a:b], plan.k_rot[a:b], plan.v[a:b], p0, p1,
                                     out=plan.out[a:b])
            ev_c = torch.cuda.Event()
            ev_c.record(s_comp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_c)
                out_host[a + p0:a + p1].copy_(plan.out[a + p0:a + p1], non_blocking=True)
        plan.comp_done[i] = ev_c
        ev_o = torch.cuda.Event()
        ev_o.record(s_out)
        plan.d2h_done[i] = ev_o
    for st in comps:
        s_out.wait_stream(st)
    plan.done = torch.cuda.Event()
    plan.done.record(s_out)
    if wait:
        cur.wait_event(plan.done)


def encode_layer_host(plan: LayerEncodePlan, q_host: torch.Tensor, k_host: torch.Tensor,
                      v_host: torch.Tensor, positions: torch.Tensor, k_pages: torch.Tensor,
                      v_pages: torch.Tensor, page_table: torch.Tensor, out_host: torch.Tensor,
                      theta: float = 10000.0, wait: bool = True) -> None:
    """Phase-1 encode of one layer from pinned host q/k/v (pre-RoPE, augmented layout) to
    pinned host out (wait: see _encode).

    positions: device int64 [rows].  Returns when every copy and kernel is queued; the
    caller synchronises (or records an event) on the current stream, which is made to wait
    on the pipeline.
    """
    def copy_in(i, r0, r1):
        plan.q[r0:r1].copy_(q_host[r0:r1], non_blocking=True)
        plan.k[r0:r1].copy_(k_host[r0:r1], non_blocking=True)
        plan.v[r0:r1].copy_(v_host[r0:r1], non_blocking=True)

    _encode(plan, copy_in, positions, k_pages, v_pages, page_table, out_host, theta, wait)


def encode_layer_host_context(plan: LayerEncodePlan, q_ctx: torch.Tensor, k_ctx: torch.Tensor,
                              v_ctx: torch.Tensor, positions: torch.Tensor, k_pages: torch.Tensor,
                              v_pages: torch.Tensor, page_table: torch.Tensor,
                              out_host: torch.Tensor, theta: float = 10000.0,
                              wait: bool = True) -> None:
    """As encode_layer_host, from pinned host q/k/v in the context layout (each distinct
    context row once, plan.set_context_layout): rows of a block cross PCIe once, anchor
    rows are replicated from the device copy of block 0.  out_host is the full augmented
    output (every encoded row)."""
    if not plan.h2d:
        raise ShapeError("call plan.set_context_layout(positions) first")
    if q_ctx.shape[0] != plan.ctx_rows:
        raise ShapeError(f"context buffers need {plan.ctx_rows} rows, got {q_ctx.shape[0]}")

    def copy_in(i, lo, hi):
        for r0, c0, m in _clip(plan.h2d[i], lo, hi):
            plan.q[r0:r0 + m].copy_(q_ctx[c0:c0 + m], non_blocking=True)
            plan.k[r0:r0 + m].copy_(k_ctx[c0:c0 + m], non_blocking=True)
            plan.v[r0:r0 + m].copy_(v_ctx[c0:c0 + m], non_blocking=True)
        for r0, src, m in _clip(plan.d2d[i], lo, hi):  # anchor rows: device copies
            plan.q[r0:r0 + m].copy_(plan.q[src:src + m], non_blocking=True)
            plan.k[r0:r0 + m].copy_(plan.k[src:src + m], non_blocking=True)
            plan.v[r0:r0 + m].copy_(plan.v[src:src + m], non_blocking=True)

    _encode(plan, copy_in, positions, k_pages, v_pages, page_table, out_host, theta, wait)
