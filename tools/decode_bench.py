"""Standalone K2 (phase-2 split-KV decode) timing at cfg2 shapes; for sweeps and ncu."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17116_b200 import ops  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--rows", type=int, default=131072)
p.add_argument("--hq", type=int, default=32)
p.add_argument("--hkv", type=int, default=8)
p.add_argument("--batch", type=int, default=1)
p.add_argument("--splits", type=int, nargs="*", default=[0])
p.add_argument("--iters", type=int, default=50)
a = p.parse_args()
dev = torch.device("cuda", 0)
d, page = 128, 128
pages = -(-a.rows // page) * a.batch
kp = ops.prng_fill((pages, a.hkv, page, d), 5, 1, 1.0, torch.bfloat16, dev)
vp = ops.prng_fill((pages, a.hkv, page, d), 6, 1, 1.0, torch.bfloat16, dev)
table = torch.arange(pages, dtype=torch.int32, device=dev).view(a.batch, -1)
q = ops.prng_fill((a.batch, 1, a.hq, d), 7, 1, 1.0, torch.bfloat16, dev)
kv_len = torch.full((a.batch,), a.rows, dtype=torch.int32, device=dev)
ws = ops.Phase2Workspace()
for sp in a.splits:
    f = lambda: ops.phase2_partial(q, kp, vp, table, kv_len, a.rows, n_splits=sp, workspace=ws)
    f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(10):
            f()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters // 10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / (a.iters // 10 * 10) * 1e3
    byts = a.batch * a.rows * a.hkv * d * 2 * 2
    print(f"splits={sp} us={us:.1f} GB/s={byts / us / 1e3:.0f} frac={byts / us / 1e3 / 6532.9:.3f}")
