"""K1 efficiency vs segment structure (cfg2 shapes): the full 8-segment cfg2 launch, one 32K
anchor-augmented segment, seven of them, and one 16K segment — alternated to cancel drift."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17116_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
hq, hkv, d = 32, 8, 128
cases = {
    "cfg2 (16K + 7x32K)": [16384] + [32768] * 7,
    "1 x 32K": [32768],
    "7 x 32K": [32768] * 7,
    "1 x 16K": [16384],
    "2 x 32K": [32768] * 2,
}
R = sum(cases["cfg2 (16K + 7x32K)"])
q = ops.prng_fill((R, hq, d), 1, 1, 1.0, torch.bfloat16, dev)
k = ops.prng_fill((R, hkv, d), 2, 1, 1.0, torch.bfloat16, dev)
v = ops.prng_fill((R, hkv, d), 3, 1, 1.0, torch.bfloat16, dev)
out = torch.empty_like(q)
res = {n: [] for n in cases}
for rep in range(3):
    for name, segs in cases.items():
        seg = [0]
        for m in segs:
            seg.append(seg[-1] + m)
        flops = sum(m * (m + 1) // 2 for m in segs) * hq * 4 * d
        rows = seg[-1]
        ops.phase1_fwd(q[:rows], k[:rows], v[:rows], seg, out=out[:rows])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 3
        e0.record()
        for _ in range(n):
            ops.phase1_fwd(q[:rows], k[:rows], v[:rows], seg, out=out[:rows])
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        res[name].append(round(flops / ms / 1e9, 1))
for name, v_ in res.items():
    print(f"{name:22s} TFLOP/s {v_}")
