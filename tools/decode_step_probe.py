"""Where a graph-captured decode step's time goes (B = 1, Llama-8B heads, one layer):
  k2        K2 alone
  append    star_kv_append alone
  app+k2    star_kv_append -> K2 (the decode step's attention)
  step      star_kv_append -> K2 -> position += 1
each captured as 20 repetitions in one CUDA graph, timed over 5 replays (µs per repetition).
Run twice to compare STAR_K2_PDL=0 / 1.  usage: python tools/decode_step_probe.py [rows...]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_17116_b200 import ops  # noqa: E402


def graph_us(fn, reps=20, replays=5):
    fn()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
        for _ in range(reps):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(replays):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * replays) * 1e3


def main():
    rows_list = [int(x) for x in sys.argv[1:]] or [4096, 16384, 131072]
    hq, hkv, d, page = 32, 8, 128, 128
    dev = torch.device("cuda", 0)
    res = {"pdl": os.environ.get("STAR_K2_PDL", "1"), "table": os.environ.get("PROBE_TABLE", "1")}
    for rows in rows_list:
        pps = -(-(rows + 4096) // page)
        kp = ops.prng_fill((pps, hkv, page, d), 1, 1, 1.0, torch.bfloat16, dev)
        vp = ops.prng_fill((pps, hkv, page, d), 2, 1, 1.0, torch.bfloat16, dev)
        table = torch.arange(pps, dtype=torch.int32, device=dev).view(1, -1)
        q = ops.prng_fill((1, hq, d), 3, 1, 1.0, torch.bfloat16, dev)
        kn = ops.prng_fill((1, hkv, d), 4, 1, 1.0, torch.bfloat16, dev)
        vn = ops.prng_fill((1, hkv, d), 5, 1, 1.0, torch.bfloat16, dev)
        pos = torch.full((1,), rows, dtype=torch.int64, device=dev)
        kv_len = torch.full((1,), rows, dtype=torch.int32, device=dev)
        ws = ops.Phase2Workspace()
        maxk = rows + 4096
        rtab = ops.RopeTable(rows, 4096, d, 10000.0, dev) if os.environ.get("PROBE_TABLE", "1") == "1" else None
        q4 = q.view(1, 1, hq, d)

        def k2():
            ops.phase2_partial(q4, kp, vp, table, kv_len, maxk, workspace=ws)

        def append():
            ops.kv_append(q, kn, vn, pos, kv_len, kp, vp, table, table=rtab)

        def app_k2():
            qr = ops.kv_append(q, kn, vn, pos, kv_len, kp, vp, table, table=rtab)
            ops.phase2_partial(qr.view(1, 1, hq, d), kp, vp, table, kv_len, maxk, workspace=ws)

        def step():
            app_k2()
            pos.add_(1)

        drope = ops.DecodeRope(rows, 4096, d, 10000.0, 1, dev)
        drope.prime(pos)

        def fused():
            ops.phase2_decode(q, kn, vn, pos, kp, vp, table, kv_len, maxk, table=rtab, workspace=ws)

        def fused_cur():
            ops.phase2_decode(q, kn, vn, pos, kp, vp, table, kv_len, maxk, table=drope,
                              workspace=ws)

        def fused_step():
            fused_cur()
            ops.decode_advance(kv_len, pos, rope=drope)

        out = {}
        for name, fn in (("k2", k2), ("append", append), ("app+k2", app_k2), ("step", step),
                         ("fused", fused), ("fused_cur", fused_cur),
                         ("fused+advance", fused_step)):
            kv_len.fill_(rows)
            out[name] = graph_us(fn)
        res[rows] = out
    print(json.dumps(res))


if __name__ == "__main__":
    main()
