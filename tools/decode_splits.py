"""Fused decode step (star_phase2_decode) per layer vs the split count, L2-cold: B = 1, Llama-8B
heads, `rows` cached rows per rank, 32 distinct caches (one per layer) in one CUDA graph + one
star_decode_advance per token.  usage: python tools/decode_splits.py [rows] [splits ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17116_b200 import ops  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
splits = [int(x) for x in sys.argv[2:]] or [0, 8, 12, 16, 18, 24, 32]
hq, hkv, d, page, L, T = 32, 8, 128, 128, 32, 16
dev = torch.device("cuda", 0)
pps = -(-(rows + 4 * T) // page)
caches = [(ops.prng_fill((pps, hkv, page, d), 2 * l + 1, 1, 1.0, torch.bfloat16, dev),
           ops.prng_fill((pps, hkv, page, d), 2 * l + 2, 1, 1.0, torch.bfloat16, dev)) for l in range(L)]
table = torch.arange(pps, dtype=torch.int32, device=dev).view(1, -1)
q = ops.prng_fill((1, hq, d), 90, 1, 1.0, torch.bfloat16, dev)
kn = ops.prng_fill((1, hkv, d), 91, 1, 1.0, torch.bfloat16, dev)
vn = ops.prng_fill((1, hkv, d), 92, 1, 1.0, torch.bfloat16, dev)
res = {"rows": rows, "us_per_layer": {}}
for ns in splits:
    kv = torch.full((1,), rows, dtype=torch.int32, device=dev)
    pos = torch.full((1,), rows, dtype=torch.int64, device=dev)
    rope = ops.DecodeRope(rows, 4 * T + 8, d, 10000.0, 1, dev)
    rope.prime(pos)
    ws = ops.Phase2Workspace()

    def step():
        for kp, vp in caches:
            ops.phase2_decode(q, kn, vn, pos, kp, vp, table, kv, rows + 4 * T, table=rope,
                              n_splits=ns, workspace=ws)
        ops.decode_advance(kv, pos, rope=rope)

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
    us = e0.elapsed_time(e1) / T / L * 1e3
    res["us_per_layer"][ns] = round(us, 2)
    del g
print(json.dumps(res))
