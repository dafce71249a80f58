"""Kernel-level operators: torch CUDA tensors in, C-ABI calls out.

Each function validates layouts, passes raw device pointers plus the current
CUDA stream to libstar_attn.so, and raises the reference's exception classes
on failure.  No operator has a CPU path: a non-CUDA tensor is an error.
"""

from __future__ import annotations

import ctypes
import os
from typing import Sequence

import torch

from . import _lib
from .errors import ConfigError, DeviceError, ShapeError

_DT = {torch.float32: _lib.STAR_F32, torch.bfloat16: _lib.STAR_BF16}


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise ConfigError(f"unsupported dtype {t.dtype}; use float32 or bfloat16") from None


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise DeviceError("star_attn operators run on CUDA tensors only (no CPU fallback)")


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _rows_view(t: torch.Tensor, name: str) -> tuple[int, int, int]:
    """[rows, heads, d] with unit inner strides; returns (rows, heads, row_stride)."""
    if t.dim() != 3:
        raise ShapeError(f"{name} must be [rows, heads, d], got shape {tuple(t.shape)}")
    if t.stride(2) != 1 or t.stride(1) != t.shape[2]:
        raise ShapeError(f"{name} must be contiguous within a row (strides {t.stride()})")
    return t.shape[0], t.shape[1], t.stride(0)


# ---------------------------------------------------------------------------- prng
def prng_fill(shape, seed: int, first: int = 1, scale: float = 1.0, dtype=torch.float32,
              device="cuda", out: torch.Tensor | None = None) -> torch.Tensor:
    """Draws first..first+n-1 of splitmix64 stream `seed` as (2u-1)*scale (ss/numerics.py:255-263).
    out: fill this contiguous tensor in place (shape/dtype/device taken from it)."""
    if out is None:
        out = torch.empty(shape, dtype=dtype, device=device)
    elif not out.is_contiguous():
        raise ShapeError("prng_fill out must be contiguous")
    _cuda(out)
    _lib.call("star_prng_fill", out.data_ptr(), dtype_code(out), out.numel(),
              int(seed) & ((1 << 64) - 1), int(first) & ((1 << 64) - 1), float(scale),
              _stream(out.device))
    return out


# ---------------------------------------------------------------------------- rope
def rope(x: torch.Tensor, positions: torch.Tensor, theta: float = 10000.0,
         out: torch.Tensor | None = None) -> torch.Tensor:
    """Adjacent-pair RoPE of x [rows, heads, d] at int64 positions [rows] (ss/numerics.py:161-180)."""
    _cuda(x, positions)
    rows, heads, xs = _rows_view(x, "x")
    if out is None:
        out = torch.empty_like(x)
    orow, oh, ys = _rows_view(out, "out")
    if (orow, oh) != (rows, heads) or out.dtype != x.dtype:
        raise ShapeError("rope out must match x")
    if positions.dtype != torch.int64 or positions.numel() != rows:
        raise ShapeError(f"{positions.numel()} positions for {rows} rows (int64 required)")
    positions = positions.contiguous()
    _lib.call("star_rope", x.data_ptr(), out.data_ptr(), dtype_code(x), rows, heads, x.shape[2],
              xs, ys, positions.data_ptr(), float(theta), _stream(x.device))
    return out


def rope_qkv(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, positions: torch.Tensor,
             theta: float = 10000.0, q_out: torch.Tensor | None = None,
             k_out: torch.Tensor | None = None, cache_rows: torch.Tensor | None = None,
             k_pages: torch.Tensor | None = None, v_pages: torch.Tensor | None = None,
             page_table: torch.Tensor | None = None):
    """Fused prologue: rotated (q, k) for K1 + own-row (rotated k, v) into pages."""
    _cuda(q, k, v, positions, cache_rows, k_pages, v_pages, page_table)
    rows, hq, qs = _rows_view(q, "q")
    rk, hkv, ks = _rows_view(k, "k")
    if rk != rows or tuple(v.shape) != tuple(k.shape) or v.stride() != k.stride():
        raise ShapeError("q/k/v rows or k/v layouts disagree")
    if not (q.dtype == k.dtype == v.dtype):
        raise ConfigError("q, k, v must share a dtype")
    if positions.dtype != torch.int64 or positions.numel() != rows:
        raise ShapeError(f"{positions.numel()} positions for {rows} rows (int64 required)")
    q_out = torch.empty_like(q) if q_out is None else q_out
    k_out = torch.empty_like(k) if k_out is None else k_out
    _, _, qos = _rows_view(q_out, "q_out")
    _, _, kos = _rows_view(k_out, "k_out")
    page_size = 0
    if cache_rows is not None:
        if cache_rows.dtype != torch.int64 or cache_rows.numel() != rows:
            raise ShapeError("cache_rows must be int64 [rows]")
        if k_pages is None or k_pages.dtype != k.dtype or k_pages.shape[1] != hkv:
            raise ShapeError("paged pool does not match k")
        page_size = k_pages.shape[2]
    _lib.call("star_rope_qkv", q.data_ptr(), k.data_ptr(), v.data_ptr(), dtype_code(q), rows, hq,
              hkv, q.shape[2], qs, ks, q_out.data_ptr(), k_out.data_ptr(), qos, kos,
              positions.contiguous().data_ptr(), float(theta), _ptr(cache_rows), _ptr(k_pages),
              _ptr(v_pages), _ptr(page_table), page_size, _stream(q.device))
    return q_out, k_out


class RopeTable:
    """cos/sin of the decode positions [pos0, pos0 + n) (star_rope_table), fp64 [n, d/2, 2]."""

    def __init__(self, pos0: int, n: int, d: int, theta: float, device):
        self.pos0, self.n, self.d, self.theta = int(pos0), int(n), int(d), float(theta)
        self.cs = torch.empty((max(self.n, 1), d // 2, 2), dtype=torch.float64, device=device)
        _lib.call("star_rope_table", self.cs.data_ptr(), self.pos0, self.n, self.d, self.theta,
                  _stream(self.cs.device))


class DecodeRope:
    """RoPE state of a fused decoder: the cos/sin table of its token budget's positions
    (RopeTable) plus `cur` — fp64 [batch, d/2, 2] cos/sin at the CURRENT positions, which
    decode_advance refreshes at the end of every token, so the next star_phase2_decode reads
    them without a dependent position load."""

    def __init__(self, pos0: int, n: int, d: int, theta: float, batch: int, device):
        self.table = RopeTable(pos0, n, d, theta, device)
        self.d, self.theta, self.batch = int(d), float(theta), int(batch)
        self.cur = torch.zeros((self.batch, d // 2, 2), dtype=torch.float64, device=device)

    def prime(self, positions: torch.Tensor) -> None:
        """cur <- cos/sin at `positions` (before the first token; no counter moves)."""
        decode_advance(positions.new_zeros(0, dtype=torch.int32), positions, add=0, rope=self,
                       inc=0)


def kv_append(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, positions: torch.Tensor,
              kv_len: torch.Tensor, k_pages: torch.Tensor, v_pages: torch.Tensor,
              page_table: torch.Tensor, theta: float = 10000.0,
              q_out: torch.Tensor | None = None, table: RopeTable | None = None) -> torch.Tensor:
    """Decode append (star_kv_append) for B = kv_len.numel() sequences of rows/B new rows each:
    rotated q returned; rotated k / raw v written at the rows each sequence's device counter
    kv_len[b] (int32) names, counters advanced — one launch, no host value, graph-capturable.
    page_table: [B, pages_per_seq] (or [pages] for B = 1).  table: precomputed cos/sin of the
    decode positions (bit-identical; positions outside it form the angle in place)."""
    _cuda(q, k, v, positions, kv_len, k_pages, v_pages, page_table)
    n, hq, qs = _rows_view(q, "q")
    rk, hkv, ks = _rows_view(k, "k")
    if rk != n or tuple(v.shape) != tuple(k.shape) or v.stride() != k.stride():
        raise ShapeError("q/k/v rows or k/v layouts disagree")
    if not (q.dtype == k.dtype == v.dtype == k_pages.dtype == v_pages.dtype):
        raise ConfigError("q, k, v and the pools must share a dtype")
    if positions.dtype != torch.int64 or positions.numel() != n:
        raise ShapeError(f"{positions.numel()} positions for {n} rows (int64 required)")
    if kv_len.dtype != torch.int32 or page_table.dtype != torch.int32:
        raise ConfigError("kv_len and page_table must be int32")
    B = kv_len.numel()
    if B < 1 or n % B:
        raise ShapeError(f"{n} rows do not split over {B} sequences")
    pt = page_table.view(1, -1) if page_table.dim() == 1 else page_table
    if pt.shape[0] != B or not pt.is_contiguous():
        raise ShapeError("page_table must be a contiguous [batch, pages_per_seq] table")
    if k_pages.dim() != 4 or k_pages.shape[1] != hkv or k_pages.shape[3] != q.shape[2]:
        raise ShapeError("paged pool does not match k")
    if table is not None and (table.d != q.shape[2] or table.theta != float(theta)):
        raise ConfigError("rope table was built for another head_dim / theta")
    q_out = torch.empty_like(q) if q_out is None else q_out
    _, _, qos = _rows_view(q_out, "q_out")
    _lib.call("star_kv_append", q.data_ptr(), k.data_ptr(), v.data_ptr(), dtype_code(q), B, n // B,
              hq, hkv, q.shape[2], qs, ks, q_out.data_ptr(), qos, positions.contiguous().data_ptr(),
              float(theta), kv_len.data_ptr(), k_pages.data_ptr(), v_pages.data_ptr(),
              pt.data_ptr(), pt.shape[1], k_pages.shape[2],
              table.cs.data_ptr() if table is not None else None,
              table.pos0 if table is not None else 0, table.n if table is not None else 0,
              _stream(q.device))
    return q_out


# ---------------------------------------------------------------------------- phase 1
def phase1_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, seg_start: Sequence[int],
               out: torch.Tensor | None = None, want_lse: bool = False, out_dtype=None,
               dedup_anchor_rows: int = 0):
    """K1: causal attention of each segment [seg_start[s], seg_start[s+1]) with itself.

    q [rows, hq, d], k/v [rows, hkv, d] (same dtype).  Returns (out, lse|None),
    lse fp32 [hq, rows] natural log.  dedup_anchor_rows > 0: rows [0, n) of every later
    segment equal segment 0's (first-block anchors) and are computed once (exact).
    """
    _cuda(q, k, v, out)
    rq, hq, qs = _rows_view(q, "q")
    rk, hkv, ks = _rows_view(k, "k")
    rv, hv, vs = _rows_view(v, "v")
    if (rk, hkv) != (rv, hv) or ks != vs:
        raise ShapeError("k and v must share shape and row stride")
    if not (q.dtype == k.dtype == v.dtype):
        raise ConfigError("q, k, v must share a dtype")
    d = q.shape[2]
    if k.shape[2] != d:
        raise ShapeError(f"q head_dim {d} != k head_dim {k.shape[2]}")
    seg = [int(x) for x in seg_start]
    if len(seg) < 1 or seg[-1] > rq or seg[-1] > rk:
        raise ShapeError("segments extend past the q/k rows")
    if out is None:
        out = torch.empty((rq, hq, d), dtype=out_dtype or q.dtype, device=q.device)
    _, _, os_ = _rows_view(out, "out")
    lse = torch.empty((hq, seg[-1]), dtype=torch.float32, device=q.device) if want_lse else None
    arr = (ctypes.c_int64 * len(seg))(*seg)
    _lib.call("star_phase1_fwd", q.data_ptr(), k.data_ptr(), v.data_ptr(), dtype_code(q),
              len(seg) - 1, arr, hq, hkv, d, qs, ks, out.data_ptr(), dtype_code(out), os_,
              _ptr(lse), int(dedup_anchor_rows), _stream(q.device))
    return out, lse


def phase1_fwd_range(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, q_begin: int, q_end: int,
                     out: torch.Tensor, lse: torch.Tensor | None = None):
    """K1 over query rows [q_begin, q_end) of one segment (row 0 at q/k/v[0]) against keys
    [0, q_end): causal_attention(q[q_begin:q_end], k[:q_end], v[:q_end], q_offset=q_begin).
    Writes out rows [q_begin, q_end) (out covers the segment) and lse [hq, >= q_end]
    columns [q_begin, q_end) when given."""
    _cuda(q, k, v, out, lse)
    rq, hq, qs = _rows_view(q, "q")
    rk, hkv, ks = _rows_view(k, "k")
    rv, hv, vs = _rows_view(v, "v")
    if (rk, hkv) != (rv, hv) or ks != vs:
        raise ShapeError("k and v must share shape and row stride")
    if not (q.dtype == k.dtype == v.dtype):
        raise ConfigError("q, k, v must share a dtype")
    if q_end > min(rq, rk) or out.shape[0] < q_end:
        raise ShapeError("query range extends past the q/k/out rows")
    _, _, os_ = _rows_view(out, "out")
    lse_stride = lse.stride(0) if lse is not None else 0
    _lib.call("star_phase1_fwd_range", q.data_ptr(), k.data_ptr(), v.data_ptr(), dtype_code(q),
              int(q_begin), int(q_end), hq, hkv, q.shape[2], qs, ks, out.data_ptr(),
              dtype_code(out), os_, _ptr(lse), lse_stride, _stream(q.device))
    return out


def phase1_fwd_check(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, seg_start: Sequence[int],
                     out_dtype=torch.float32, want_lse: bool = True):
    """Check mode of phase1_fwd: the fp32 CUDA-core kernel for any input dtype."""
    _cuda(q, k, v)
    rq, hq, qs = _rows_view(q, "q")
    rk, hkv, ks = _rows_view(k, "k")
    if tuple(v.shape) != tuple(k.shape) or v.stride() != k.stride():
        raise ShapeError("k and v must share shape and row stride")
    d = q.shape[2]
    seg = [int(x) for x in seg_start]
    if seg[-1] > rq or seg[-1] > rk:
        raise ShapeError("segments extend past the q/k rows")
    out = torch.empty((rq, hq, d), dtype=out_dtype, device=q.device)
    lse = torch.empty((hq, seg[-1]), dtype=torch.float32, device=q.device) if want_lse else None
    arr = (ctypes.c_int64 * len(seg))(*seg)
    _lib.call("star_phase1_fwd_check", q.data_ptr(), k.data_ptr(), v.data_ptr(), dtype_code(q),
              len(seg) - 1, arr, hq, hkv, d, qs, ks, out.data_ptr(), dtype_code(out), hq * d,
              _ptr(lse), _stream(q.device))
    return out, lse


def attention_dense(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, q_offset: int = 0,
                    mask: str = "causal", want_lse: bool = True):
    """Masked attention of q [lq, hq, d] vs k/v [lk, hkv, d]; mask "causal" | "full"."""
    _cuda(q, k, v)
    lq, hq, qs = _rows_view(q, "q")
    lk, hkv, ks = _rows_view(k, "k")
    if tuple(v.shape) != tuple(k.shape) or v.stride() != k.stride():
        raise ShapeError("k and v must share shape and strides")
    if q.shape[2] != k.shape[2]:
        raise ShapeError(f"q cols {q.shape[2]} != k cols {k.shape[2]}")
    if mask not in ("causal", "full"):
        raise ConfigError(f"unknown mask kind {mask!r}")
    d = q.shape[2]
    out = torch.empty((lq, hq, d), dtype=q.dtype, device=q.device)
    lse = torch.empty((hq, lq), dtype=torch.float32, device=q.device) if want_lse else None
    _lib.call("star_attention_dense", q.data_ptr(), k.data_ptr(), v.data_ptr(), dtype_code(q), lq,
              lk, int(q_offset), 1 if mask == "causal" else 0, hq, hkv, d, qs, ks,
              out.data_ptr(), hq * d, _ptr(lse), _stream(q.device))
    return out, lse


# ---------------------------------------------------------------------------- paged KV
def kv_write(k: torch.Tensor, v: torch.Tensor, k_pages: torch.Tensor, v_pages: torch.Tensor,
             page_table: torch.Tensor, dst_row0: int) -> None:
    """Write rows of k/v [n, hkv, d] to logical rows [dst_row0, dst_row0+n) of a paged cache."""
    _cuda(k, v, k_pages, v_pages, page_table)
    n, hkv, ks = _rows_view(k, "k")
    if tuple(v.shape) != tuple(k.shape) or v.stride() != k.stride():
        raise ShapeError("k and v must share shape and strides")
    if k_pages.dim() != 4 or k_pages.shape[1] != hkv or k_pages.shape[3] != k.shape[2]:
        raise ShapeError(f"pool shape {tuple(k_pages.shape)} does not match k {tuple(k.shape)}")
    if k_pages.dtype != k.dtype:
        raise ConfigError("pool dtype must match k/v")
    page_size = k_pages.shape[2]
    if (dst_row0 + n + page_size - 1) // page_size > page_table.numel():
        raise ShapeError("page table too short for the written rows")
    _lib.call("star_kv_write", k.data_ptr(), v.data_ptr(), dtype_code(k), n, hkv, k.shape[2], ks,
              k_pages.data_ptr(), v_pages.data_ptr(), page_table.data_ptr(), page_size,
              int(dst_row0), _stream(k.device))


def kv_read(k_pages: torch.Tensor, v_pages: torch.Tensor, page_table: torch.Tensor, row0: int,
            n_rows: int):
    _cuda(k_pages, v_pages, page_table)
    _, hkv, page_size, d = k_pages.shape
    k = torch.empty((n_rows, hkv, d), dtype=k_pages.dtype, device=k_pages.device)
    v = torch.empty_like(k)
    _lib.call("star_kv_read", k_pages.data_ptr(), v_pages.data_ptr(), dtype_code(k_pages),
              page_table.data_ptr(), page_size, int(row0), int(n_rows), hkv, d, k.data_ptr(),
              v.data_ptr(), _stream(k.device))
    return k, v


# ---------------------------------------------------------------------------- phase 2
class Phase2Workspace:
    """Reusable device workspace for the split partials (sized on demand).

    Zero-initialised.  Its header holds the bf16 kernel's per-(sequence, kv head) arrival
    counters (re-armed to zero by every launch) and word-mode epochs (advanced by every
    launch); the library re-zeroes it itself when a call changes the shape or fix-up mode."""

    def __init__(self):
        self.buf: torch.Tensor | None = None

    def get(self, nbytes: int, device) -> int | None:
        if nbytes <= 0:
            return None
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != torch.device(device):
            self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        return self.buf.data_ptr()


# default workspaces, one per (device, stream): the split-arrival counters and word-mode
# epochs in a workspace are only safe for stream-ordered launches, so two streams never share one
_default_ws: dict = {}


def _phase2_args(q, k_pages, v_pages, page_table, kv_len, max_kv_len, own_tail, n_splits, out,
                 lse, workspace, qshape=None):
    """Validated argument tuple of star_phase2_partial[_push] (everything but the stream).
    qshape: (B, lq, hq, d) of a q whose layout the caller validated (the fused decode's
    strided pre-RoPE rows)."""
    _cuda(q, k_pages, v_pages, page_table, kv_len)
    if qshape is None:
        if q.dim() != 4 or not q.is_contiguous():
            raise ShapeError("q must be a contiguous [batch, lq, hq, d] tensor")
        qshape = tuple(q.shape)
    B, lq, hq, d = qshape
    if k_pages.dim() != 4 or k_pages.shape != v_pages.shape:
        raise ShapeError("k/v pools must be [num_pages, hkv, page_size, d]")
    _, hkv, page_size, dk = k_pages.shape
    if dk != d:
        raise ShapeError(f"q cols {d} != cache cols {dk}")
    if page_table.dtype != torch.int32 or kv_len.dtype != torch.int32:
        raise ConfigError("page_table and kv_len must be int32")
    if page_table.dim() == 1:
        page_table = page_table.view(1, -1)
    if page_table.shape[0] != B or kv_len.numel() != B:
        raise ShapeError("page_table / kv_len batch mismatch")
    page_table = page_table.contiguous()
    pps = page_table.shape[1]
    if (max_kv_len + page_size - 1) // page_size > pps:
        raise ShapeError("page table shorter than max_kv_len")
    lib = _lib.load()
    if n_splits <= 0:
        # (the tensor-core kernel runs > 16 query rows per kv head as 64-row blocks; one wave
        # counts each block, as star_phase2_partial does for n_splits = 0)
        qrows = (hq // hkv) * lq
        qe = (q.dtype == torch.bfloat16 and d == 128 and 16 < qrows <= 128 and page_size % 64 == 0
              and os.environ.get("STAR_K2_QE", "1")[:1] != "0")  # tcgen05 query encode: 1 tile
        n_rb = 1 if (qrows <= 16 or qe) else -(-qrows // 64)
        n_splits = lib.star_phase2_auto_splits(B, hkv * n_rb, int(max_kv_len), page_size)
    if out is None:
        out = torch.empty((B, lq, hq, d), dtype=torch.float32, device=q.device)
    if lse is None:
        lse = torch.empty((B, lq, hq), dtype=torch.float32, device=q.device)
    nbytes = lib.star_phase2_workspace_bytes(B, lq, hq, d, n_splits)
    ws = workspace or _default_ws.setdefault((q.device, _stream(q.device)), Phase2Workspace())
    args = (q.data_ptr(), dtype_code(q), B, lq, hq, hkv, d, k_pages.data_ptr(), v_pages.data_ptr(),
            dtype_code(k_pages), k_pages.shape[0], page_table.data_ptr(), pps, page_size,
            kv_len.data_ptr(), int(max_kv_len), int(own_tail), out.data_ptr(), lse.data_ptr(), int(n_splits),
            ws.get(nbytes, q.device))
    return args, out, lse


def phase2_partial(q: torch.Tensor, k_pages: torch.Tensor, v_pages: torch.Tensor,
                   page_table: torch.Tensor, kv_len: torch.Tensor, max_kv_len: int,
                   own_tail: int = 0, n_splits: int = 0, out: torch.Tensor | None = None,
                   lse: torch.Tensor | None = None, workspace: Phase2Workspace | None = None):
    """K2: partial attention of q [B, lq, hq, d] vs each sequence's paged cache.

    Returns fp32 (out [B, lq, hq, d], lse [B, lq, hq]).
    """
    args, out, lse = _phase2_args(q, k_pages, v_pages, page_table, kv_len, max_kv_len, own_tail,
                                  n_splits, out, lse, workspace)
    _lib.call("star_phase2_partial", *args, _stream(q.device))
    return out, lse


def _decode_args(q, k, v, positions, append, theta, table, k_pages, v_pages, page_table, kv_len,
                 max_kv_len, n_splits, out, lse, workspace):
    """Validated argument tuple of star_phase2_decode[_exchange] (everything but the stream)."""
    _cuda(q, positions, k_pages, v_pages, page_table, kv_len)
    if q.dim() != 3 or q.stride(2) != 1 or q.stride(1) != q.shape[2]:
        raise ShapeError("q must be [batch, hq, d] with packed heads")
    B, hq, d = q.shape
    if append:
        _cuda(k, v)
        if k.dim() != 3 or tuple(v.shape) != tuple(k.shape) or v.stride() != k.stride():
            raise ShapeError("k / v must be [batch, hkv, d] with one layout")
        if k.stride(2) != 1 or k.stride(1) != k.shape[2]:
            raise ShapeError("k / v heads must be packed")
    if q.dtype != torch.bfloat16 or k_pages.dtype != torch.bfloat16 or (append and k.dtype != torch.bfloat16):
        raise ConfigError("the fused decode step is bf16")
    if positions.dtype != torch.int64 or positions.numel() != B:
        raise ShapeError(f"{positions.numel()} positions for batch {B} (int64 required)")
    cur = None
    if isinstance(table, DecodeRope):
        if table.batch != B:
            raise ShapeError(f"DecodeRope holds {table.batch} sequences, batch is {B}")
        cur, table = table.cur, table.table
    if table is not None and (table.d != d or table.theta != float(theta)):
        raise ConfigError("rope table was built for another head_dim / theta")
    (pargs, out, lse) = _phase2_args(q, k_pages, v_pages, page_table, kv_len, max_kv_len, 0,
                                     n_splits, out, lse, workspace, qshape=(B, 1, hq, d))
    _, _, _, _, _, hkv, _, kp, vp, _, num_pages, pt, pps, page_size, kl, mk, _, o, l, ns, ws = pargs
    args = (q.data_ptr(), k.data_ptr() if append else None, v.data_ptr() if append else None,
            1 if append else 0, q.stride(0), k.stride(0) if append else hkv * d,
            positions.contiguous().data_ptr(), float(theta),
            table.cs.data_ptr() if table is not None else None,
            table.pos0 if table is not None else 0, table.n if table is not None else 0,
            cur.data_ptr() if cur is not None else None,
            B, hq, hkv, d, kp, vp, num_pages, pt, pps, page_size, kl, mk, o, l, ns, ws)
    return args, out, lse


def phase2_decode(q: torch.Tensor, k: torch.Tensor | None, v: torch.Tensor | None,
                  positions: torch.Tensor, k_pages: torch.Tensor, v_pages: torch.Tensor,
                  page_table: torch.Tensor, kv_len: torch.Tensor, max_kv_len: int,
                  theta: float = 10000.0, table: "RopeTable | DecodeRope | None" = None,
                  append: bool = True,
                  n_splits: int = 0, out: torch.Tensor | None = None,
                  lse: torch.Tensor | None = None, workspace: Phase2Workspace | None = None):
    """Fused decode step of one layer (star_phase2_decode): RoPE of the token's PRE-RoPE q
    [B, hq, d] inside K2 and, with append, its rotated k / raw v [B, hkv, d] written at row
    kv_len[b] of each paged cache by the K2 CTA that streams that row — then attention over
    kv_len[b] + 1 rows.  One launch instead of kv_append + phase2_partial, bit-identical to
    them.  kv_len is NOT advanced (decode_advance once per token).
    Returns fp32 (out [B, 1, hq, d], lse [B, 1, hq])."""
    args, out, lse = _decode_args(q, k, v, positions, append, theta, table, k_pages, v_pages,
                                  page_table, kv_len, max_kv_len, n_splits, out, lse, workspace)
    _lib.call("star_phase2_decode", *args, _stream(q.device))
    return out, lse


def phase2_decode_exchange(q, k, v, positions, k_pages, v_pages, page_table, kv_len,
                           max_kv_len, boxes: Sequence[int], cap_rows: int, cap_groups: int,
                           rank: int, theta: float = 10000.0, table: RopeTable | None = None,
                           append: bool = True, n_splits: int = 0,
                           workspace: Phase2Workspace | None = None):
    """phase2_decode with the fused peer exchange (phase2_exchange): returns the merged
    fp32 (out [B, 1, hq, d], lse [B, 1, hq]) on every rank."""
    args, out, lse = _decode_args(q, k, v, positions, append, theta, table, k_pages, v_pages,
                                  page_table, kv_len, max_kv_len, n_splits, None, None, workspace)
    _lib.call("star_phase2_decode_exchange", *args, _box_array(boxes), len(boxes), int(cap_rows),
              int(cap_groups), int(rank), _stream(q.device))
    return out, lse


def decode_advance(kv_len: torch.Tensor, positions: torch.Tensor | None, add: int = 1,
                   rope: DecodeRope | None = None, inc: int = 1) -> None:
    """End of a fused decode token (star_decode_advance, one launch): every int32 counter in
    kv_len += add, every int64 position += inc and, with `rope`, rope.cur <- cos/sin at the new
    positions."""
    _cuda(kv_len)
    if kv_len.dtype != torch.int32 or not kv_len.is_contiguous():
        raise ConfigError("kv_len must be contiguous int32")
    if positions is not None:
        _cuda(positions)
        if positions.dtype != torch.int64 or not positions.is_contiguous():
            raise ConfigError("positions must be contiguous int64")
    if rope is not None and (positions is None or positions.numel() != rope.batch):
        raise ShapeError("rope refresh needs one position per sequence")
    tab = rope.table if rope is not None else None
    _lib.call("star_decode_advance", kv_len.data_ptr(), kv_len.numel(), int(add),
              positions.data_ptr() if positions is not None else None,
              positions.numel() if positions is not None else 0, int(inc),
              rope.cur.data_ptr() if rope is not None else None,
              tab.cs.data_ptr() if tab is not None else None, tab.pos0 if tab is not None else 0,
              tab.n if tab is not None else 0, rope.d if rope is not None else 0,
              rope.theta if rope is not None else 0.0, _stream(kv_len.device))


# ---------------------------------------------------------------- peer exchange (fused C1)
def exchange_box_bytes(world: int, cap_rows: int, cap_groups: int, d: int) -> int:
    n = _lib.load().star_exchange_box_bytes(world, cap_rows, cap_groups, d)
    _lib.check(0 if n > 0 else int(n))
    return int(n)


def ipc_get_handle(t: torch.Tensor) -> tuple[bytes, int]:
    """(CUDA IPC handle of t's allocation, t's byte offset inside it)."""
    _cuda(t)
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64(0)
    _lib.call("star_ipc_get_handle", t.data_ptr(), h, ctypes.byref(off))
    return h.raw, int(off.value)


def ipc_open_handle(handle: bytes, offset: int) -> int:
    """Map another process's allocation; returns the device address of (base + offset)."""
    ptr = ctypes.c_void_p(0)
    _lib.call("star_ipc_open_handle", ctypes.create_string_buffer(bytes(handle), 64), int(offset),
              ctypes.byref(ptr))
    return int(ptr.value)


def ipc_close_handle(ptr: int, offset: int) -> None:
    _lib.call("star_ipc_close_handle", ptr, int(offset))


def _box_array(boxes: Sequence[int]):
    return (ctypes.c_void_p * len(boxes))(*boxes)


def phase2_partial_push(q: torch.Tensor, k_pages: torch.Tensor, v_pages: torch.Tensor,
                        page_table: torch.Tensor, kv_len: torch.Tensor, max_kv_len: int,
                        boxes: Sequence[int], cap_rows: int, cap_groups: int, rank: int,
                        own_tail: int = 0, n_splits: int = 0,
                        workspace: Phase2Workspace | None = None) -> None:
    """K2 whose epilogue stores each group's final partial into slot `rank` of every box
    (device pointers `boxes`, one per rank) and releases the group's flag for the exchange
    in flight (epochs are counted on the device, csrc/exchange.cuh)."""
    args, _, _ = _phase2_args(q, k_pages, v_pages, page_table, kv_len, max_kv_len, own_tail,
                              n_splits, None, None, workspace)
    _lib.call("star_phase2_partial_push", *args, _box_array(boxes), len(boxes), int(cap_rows),
              int(cap_groups), int(rank), _stream(q.device))


def phase2_exchange(q: torch.Tensor, k_pages: torch.Tensor, v_pages: torch.Tensor,
                    page_table: torch.Tensor, kv_len: torch.Tensor, max_kv_len: int,
                    boxes: Sequence[int], cap_rows: int, cap_groups: int, rank: int,
                    own_tail: int = 0, n_splits: int = 0,
                    workspace: Phase2Workspace | None = None):
    """One layer's whole phase-2 exchange: this rank's partial pushed to every box and every
    rank's partials merged (one kernel when the K2 grid is co-resident, else K2 + K3x).
    Returns fp32 (out [B, lq, hq, d], lse [B, lq, hq])."""
    args, out, lse = _phase2_args(q, k_pages, v_pages, page_table, kv_len, max_kv_len, own_tail,
                                  n_splits, None, None, workspace)
    _lib.call("star_phase2_exchange", *args, _box_array(boxes), len(boxes), int(cap_rows),
              int(cap_groups), int(rank), _stream(q.device))
    return out, lse


def exchange_push(out: torch.Tensor, lse: torch.Tensor, batch: int, lq: int, hq: int, hkv: int,
                  boxes: Sequence[int], cap_rows: int, cap_groups: int, rank: int) -> None:
    """Deliver a partial already in device memory (fp32 out [B*lq*hq, d], lse) to every box."""
    _cuda(out, lse)
    if out.dtype != torch.float32 or lse.dtype != torch.float32:
        raise ConfigError("partials must be fp32")
    out, lse = out.contiguous(), lse.contiguous()
    d = out.shape[-1]
    if out.numel() != batch * lq * hq * d or lse.numel() != batch * lq * hq:
        raise ShapeError("partial does not match batch x lq x hq")
    _lib.call("star_exchange_push", out.data_ptr(), lse.data_ptr(), batch, lq, hq, hkv, d,
              _box_array(boxes), len(boxes), int(cap_rows), int(cap_groups), int(rank),
              _stream(out.device))


def exchange_merge(box: int, world: int, cap_rows: int, cap_groups: int, batch: int, lq: int,
                   hq: int, hkv: int, d: int, device, out_dtype=torch.float32):
    """K3x: wait for every rank's partial of the exchange in flight in `box`, merge them in
    ascending rank order and advance the box's epoch.
    Returns (out [batch*lq*hq, d], lse [batch*lq*hq])."""
    rows = batch * lq * hq
    out = torch.empty((rows, d), dtype=out_dtype, device=device)
    lse = torch.empty((rows,), dtype=torch.float32, device=device)
    _lib.call("star_exchange_merge", box, world, int(cap_rows), int(cap_groups), batch, lq, hq,
              hkv, d, out.data_ptr(), _DT[out_dtype], lse.data_ptr(), _stream(device))
    return out, lse


def merge(outs: torch.Tensor, lses: torch.Tensor, out_dtype=torch.float32):
    """K3: merge partials outs [P, rows, d], lses [P, rows] in ascending part order."""
    _cuda(outs, lses)
    if outs.dtype != torch.float32 or lses.dtype != torch.float32:
        raise ConfigError("partials must be fp32")
    if outs.dim() != 3 or lses.shape != outs.shape[:2]:
        raise ShapeError("outs [P, rows, d] and lses [P, rows] required")
    outs, lses = outs.contiguous(), lses.contiguous()
    P, rows, d = outs.shape
    out = torch.empty((rows, d), dtype=out_dtype, device=outs.device)
    lse = torch.empty((rows,), dtype=torch.float32, device=outs.device)
    _lib.call("star_merge", outs.data_ptr(), lses.data_ptr(), P, rows, d, out.data_ptr(),
              _DT[out_dtype], lse.data_ptr(), _stream(outs.device))
    return out, lse


def packed_partial(rows: int, d: int, device) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """One fp32 buffer [rows*d out | rows lse] plus (out, lse) views into it: K2 writes its
    partial straight into the wire format of the single all-gather (dist.gather_merge)."""
    buf = torch.empty(rows * (d + 1), dtype=torch.float32, device=device)
    return buf, buf[:rows * d].view(rows, d), buf[rows * d:]


def merge_packed(parts: torch.Tensor, rows: int, d: int, out_dtype=torch.float32):
    """K3 over all-gathered packed partials parts [P, rows*(d+1)] (ascending part order)."""
    _cuda(parts)
    if parts.dtype != torch.float32:
        raise ConfigError("partials must be fp32")
    if parts.dim() != 2 or parts.shape[1] != rows * (d + 1):
        raise ShapeError("packed partials must be [P, rows*(d+1)]")
    parts = parts.contiguous()
    P = parts.shape[0]
    out = torch.empty((rows, d), dtype=out_dtype, device=parts.device)
    lse = torch.empty((rows,), dtype=torch.float32, device=parts.device)
    base = parts.data_ptr()
    _lib.call("star_merge_strided", base, rows * (d + 1), base + rows * d * 4, rows * (d + 1), P,
              rows, d, out.data_ptr(), _DT[out_dtype], lse.data_ptr(), _stream(parts.device))
    return out, lse


def debug_umma_gemm(a: torch.Tensor, b: torch.Tensor, b_mn_major: bool = False,
                    a_tmem: bool = False) -> torch.Tensor:
    """C = A . B^T on one tcgen05 CTA (descriptor self-test); a [128, K], b [128, K] or [K, 128]."""
    _cuda(a, b)
    K = a.shape[1]
    c = torch.empty((128, 128), dtype=torch.float32, device=a.device)
    _lib.call("star_debug_umma_gemm", a.contiguous().data_ptr(), b.contiguous().data_ptr(),
              c.data_ptr(), K, (1 if b_mn_major else 0) | (2 if a_tmem else 0), _stream(a.device))
    return c
