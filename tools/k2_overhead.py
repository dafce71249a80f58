"""Fixed cost of a chained K2 launch: µs per layer of 32 graph-captured launches (one cache per
layer) vs cached rows, for K2 alone and the fused decode step, plus the floor of 32 chained
tiny kernels (star_decode_advance).  A linear fit over rows separates the per-launch overhead
from the streaming rate.  Launch knobs (STAR_K2_PDL, STAR_K2_COOP, STAR_K2_FIXUP) are read
once per process: run once per setting.
usage: python tools/k2_overhead.py [rows ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("STAR_LIB_PATH"):  # A/B against another build
    from paper_2411_17116_b200 import _lib  # noqa: E402
    _lib.LIB_PATH = os.environ["STAR_LIB_PATH"]
from paper_2411_17116_b200 import ops  # noqa: E402

rows_list = [int(x) for x in sys.argv[1:]] or [256, 1024, 4096, 16384, 32768]
hq, hkv, d, page, L, T = 32, 8, 128, 128, 32, 16
dev = torch.device("cuda", 0)


def graph_us(step):
    step()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
        step()
    torch.cuda.current_stream().wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(T):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / T / L * 1e3


env = {k: os.environ[k] for k in os.environ if k.startswith("STAR_K2") or k == "STAR_LIB_PATH"}
res = {"env": env, "rows": rows_list, "k2": [], "decode": []}
q = ops.prng_fill((1, hq, d), 90, 1, 1.0, torch.bfloat16, dev)
kn = ops.prng_fill((1, hkv, d), 91, 1, 1.0, torch.bfloat16, dev)
vn = ops.prng_fill((1, hkv, d), 92, 1, 1.0, torch.bfloat16, dev)
for rows in rows_list:
    pps = -(-(rows + 4 * T + 8) // page)
    caches = [(ops.prng_fill((pps, hkv, page, d), 2 * l + 1, 1, 1.0, torch.bfloat16, dev),
               ops.prng_fill((pps, hkv, page, d), 2 * l + 2, 1, 1.0, torch.bfloat16, dev))
              for l in range(L)]
    table = torch.arange(pps, dtype=torch.int32, device=dev).view(1, -1)
    kv = torch.full((1,), rows, dtype=torch.int32, device=dev)
    pos = torch.full((1,), rows, dtype=torch.int64, device=dev)
    rope = ops.DecodeRope(rows, 4 * T + 8, d, 10000.0, 1, dev)
    rope.prime(pos)
    ws = ops.Phase2Workspace()
    maxk = rows + 4 * T + 8

    def k2():
        for kp, vp in caches:
            ops.phase2_partial(q.view(1, 1, hq, d), kp, vp, table, kv, maxk, workspace=ws)

    def dec():
        for kp, vp in caches:
            ops.phase2_decode(q, kn, vn, pos, kp, vp, table, kv, maxk, table=rope, workspace=ws)
        ops.decode_advance(kv, pos, rope=rope)

    res["k2"].append(round(graph_us(k2), 2))
    kv.fill_(rows)
    pos.fill_(rows)
    rope.prime(pos)
    res["decode"].append(round(graph_us(dec), 2))
    del caches
    torch.cuda.empty_cache()

kv = torch.zeros((L,), dtype=torch.int32, device=dev)
pos = torch.zeros((1,), dtype=torch.int64, device=dev)
res["tiny_kernel_floor"] = round(graph_us(lambda: [ops.decode_advance(kv[i:i + 1], pos)
                                                    for i in range(L)]), 2)
x = np.array(rows_list, dtype=np.float64)
for k in ("k2", "decode"):
    y = np.array(res[k])
    slope, icpt = np.polyfit(x, y, 1)
    res[k + "_fit"] = {"fixed_us": round(float(icpt), 2),
                       "GBps": round(float(hkv * d * 4 / slope / 1e3), 1)}
print(json.dumps(res))
