"""Small launches of every product kernel for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): K1 (tcgen05, both head dims, dedup, query range), the fp32 check
kernels, K2 decode (word-mode split fold), K2q query encode, the fused one-kernel peer
exchange and the K2-push + K3x pair (local boxes), K3 merge, the decode append, the fused
decode step (star_phase2_decode[_exchange], star_decode_advance), RoPE, page write/read.  usage: compute-sanitizer --tool X python tools/sanitize_cases.py [--serial]

--serial: every split-KV launch with ONE split per (sequence, kv head), so no CTA spin-waits on
another (racecheck / synccheck run CTAs one at a time, under which the co-resident word-mode
fold and the one-kernel exchange cannot make progress); the exchanges then take the
K2-push + K3x form."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_17116_b200 import dist as D  # noqa: E402
from paper_2411_17116_b200 import ops  # noqa: E402


def main():
    serial = "--serial" in sys.argv
    ns = 1 if serial else 0  # n_splits for the split-KV launches
    dev = torch.device("cuda", 0)
    bf = torch.bfloat16
    # K1
    for d, hq, hkv in ((128, 8, 2), (64, 4, 4)):
        seg = [0, 256, 256 + 384]
        q = ops.prng_fill((seg[-1], hq, d), 1, 1, 1.0, bf, dev)
        k = ops.prng_fill((seg[-1], hkv, d), 2, 1, 1.0, bf, dev)
        v = ops.prng_fill((seg[-1], hkv, d), 3, 1, 1.0, bf, dev)
        ops.phase1_fwd(q, k, v, seg, want_lse=True)
        ops.phase1_fwd_check(q, k, v, seg)
    k[256:384] = k[:128]
    v[256:384] = v[:128]
    q[256:384] = q[:128]
    ops.phase1_fwd(q, k, v, seg, dedup_anchor_rows=128)
    out = torch.empty((384, hq, d), dtype=bf, device=dev)
    ops.phase1_fwd_range(q[256:].contiguous(), k[256:].contiguous(), v[256:].contiguous(), 128, 384,
                         out=out)
    # paged cache + RoPE + append
    hq, hkv, d, page = 32, 8, 128, 64
    rows = 3000
    pages = -(-(rows + 64) // page)
    kp = torch.zeros((pages, hkv, page, d), dtype=bf, device=dev)
    vp = torch.zeros_like(kp)
    table = torch.arange(pages, dtype=torch.int32, device=dev)
    kk = ops.prng_fill((rows, hkv, d), 4, 1, 1.0, bf, dev)
    vv = ops.prng_fill((rows, hkv, d), 5, 1, 1.0, bf, dev)
    ops.kv_write(kk, vv, kp, vp, table, 0)
    ops.kv_read(kp, vp, table, 0, rows)
    pos = torch.arange(rows, dtype=torch.int64, device=dev)
    ops.rope(kk, pos)
    kv_len = torch.tensor([rows], dtype=torch.int32, device=dev)
    qn = ops.prng_fill((1, hq, d), 6, 1, 1.0, bf, dev)
    kn = ops.prng_fill((1, hkv, d), 7, 1, 1.0, bf, dev)
    ops.kv_append(qn, kn, kn, torch.tensor([rows], dtype=torch.int64, device=dev), kv_len, kp, vp,
                  table, table=ops.RopeTable(rows, 8, d, 10000.0, dev))
    n = rows + 1
    # K2 decode (word-mode fold) and K2q query encode
    q1 = ops.prng_fill((1, 1, hq, d), 8, 1, 1.0, bf, dev)
    ops.phase2_partial(q1, kp, vp, table.view(1, -1), kv_len, n, n_splits=ns)
    q32 = ops.prng_fill((1, 32, hq, d), 9, 1, 1.0, bf, dev)
    ops.phase2_partial(q32, kp, vp, table.view(1, -1), kv_len, n, own_tail=32, n_splits=ns)
    ops.phase2_partial(q1.float(), kp.float(), vp.float(), table.view(1, -1), kv_len, n,
                       n_splits=ns)
    # exchanges: one-kernel (1 rank) and push + K3x (2 ranks' boxes in this process)
    ex1 = D.local_peer_exchanges(1, hq, hkv, d, dev)[0]
    ex1.exchange(q1, kp, vp, table.view(1, -1), kv_len, n, n_splits=ns)
    exs = D.local_peer_exchanges(2, hq, hkv, d, dev)
    for r in range(2):
        exs[r].push_partial(q1, kp, vp, table.view(1, -1), kv_len, n, n_splits=ns)
    for r in range(2):
        exs[r].merge(1, 1, hq, hkv)
    o, s = ops.phase2_partial(q1, kp, vp, table.view(1, -1), kv_len, n, n_splits=ns)
    ops.merge(torch.stack([o.view(hq, d)] * 3), torch.stack([s.view(hq)] * 3))
    # fused decode (RoPE + append inside K2), with the current-position cos/sin, the counter
    # advance, and the fused decode through the one-kernel exchange (1 rank)
    posn = torch.tensor([n], dtype=torch.int64, device=dev)
    rope = ops.DecodeRope(n, 8, d, 10000.0, 1, dev)
    rope.prime(posn)
    ops.phase2_decode(qn, kn, kn, posn, kp, vp, table.view(1, -1), kv_len, n + 1, table=rope,
                      n_splits=ns)
    ops.phase2_decode(qn, None, None, posn, kp, vp, table.view(1, -1), kv_len, n + 1, table=rope,
                      append=False, n_splits=ns)
    ex1.decode_exchange(qn, kn, kn, posn, kp, vp, table.view(1, -1), kv_len, n + 1, 10000.0, rope,
                        n_splits=ns)
    ops.decode_advance(kv_len, posn, rope=rope)
    torch.cuda.synchronize()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
