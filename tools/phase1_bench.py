"""Standalone K1 timing at cfg2 (or cfg4) shapes — tuning knob sweeps (e.g. STAR_K1_POLY)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("STAR_LIB_PATH"):  # A/B against another build
    from paper_2411_17116_b200 import _lib  # noqa: E402
    _lib.LIB_PATH = os.environ["STAR_LIB_PATH"]
from paper_2411_17116_b200 import ops  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--L", type=int, default=131072)
p.add_argument("--b", type=int, default=16384)
p.add_argument("--hq", type=int, default=32)
p.add_argument("--hkv", type=int, default=8)
p.add_argument("--iters", type=int, default=5)
p.add_argument("--save", default=None, help="write the output (for bit-exact A/B checks)")
a = p.parse_args()
dev = torch.device("cuda", 0)
n = -(-a.L // a.b)
seg = [0]
for i in range(n):
    seg.append(seg[-1] + min(a.b, a.L - i * a.b) + (a.b if i else 0))
R = seg[-1]
q = ops.prng_fill((R, a.hq, 128), 1, 1, 1.0, torch.bfloat16, dev)
k = ops.prng_fill((R, a.hkv, 128), 2, 1, 1.0, torch.bfloat16, dev)
v = ops.prng_fill((R, a.hkv, 128), 3, 1, 1.0, torch.bfloat16, dev)
out = torch.empty_like(q)
pairs = sum((seg[i + 1] - seg[i]) * (seg[i + 1] - seg[i] + 1) // 2 for i in range(n))
flops = pairs * a.hq * 4 * 128
for _ in range(2):
    ops.phase1_fwd(q, k, v, seg, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402

with ClockSampler(0) as clk:
    e0.record()
    for _ in range(a.iters):
        ops.phase1_fwd(q, k, v, seg, out=out)
    e1.record()
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
mhz = clk.summary()["sm_mhz"] or float("nan")
knobs = " ".join(f"{k}={os.environ[k]}" for k in sorted(os.environ) if k.startswith("STAR_K1_"))
print(f"{knobs or 'defaults'} ms={ms:.2f} TFLOP/s={flops / ms / 1e9:.1f} sm_mhz={mhz:.0f} "
      f"Mclk={ms * mhz / 1e3:.2f} flop/clk/SM={flops / (ms * 1e-3 * mhz * 1e6) / 148:.0f}")
if a.save:  # every 61st row (all heads): enough for a bit-exact A/B without GBs on the host
    torch.save(out[::61].cpu(), a.save)
