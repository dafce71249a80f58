"""Fused prologue (star_rope_qkv) at cfg2 shapes: 245,760 augmented rows, 32 q / 8 kv heads,
d = 128, own rows into a paged cache; us per launch and GB/s of its bytes (q, k, v read; q, k
rotated and own-row k, v pages written).  STAR_LIB_PATH=... times another build (A/B).
With --check FILE: save (or, if FILE exists, compare bit for bit) a strided sample of outputs."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("STAR_LIB_PATH"):
    from paper_2411_17116_b200 import _lib  # noqa: E402
    _lib.LIB_PATH = os.environ["STAR_LIB_PATH"]
from paper_2411_17116_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
R, hq, hkv, d, own, page = 245760, 32, 8, 128, 131072, 128
q = ops.prng_fill((R, hq, d), 1, 1, 1.0, torch.bfloat16, dev)
k = ops.prng_fill((R, hkv, d), 2, 1, 1.0, torch.bfloat16, dev)
v = ops.prng_fill((R, hkv, d), 3, 1, 1.0, torch.bfloat16, dev)
pos = torch.arange(R, dtype=torch.int64, device=dev) % 131072
cache_rows = torch.full((R,), -1, dtype=torch.int64, device=dev)
cache_rows[R - own:] = torch.arange(own, device=dev)
kp = torch.zeros((own // page, hkv, page, d), dtype=torch.bfloat16, device=dev)
vp = torch.zeros_like(kp)
table = torch.randperm(own // page, generator=torch.Generator().manual_seed(0)).to(torch.int32).to(dev)
qo, ko = torch.empty_like(q), torch.empty_like(k)
f = lambda: ops.rope_qkv(q, k, v, pos, q_out=qo, k_out=ko, cache_rows=cache_rows, k_pages=kp,  # noqa
                         v_pages=vp, page_table=table)
for _ in range(3):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    f()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
nbytes = 2 * (2 * R * hq * d + 3 * R * hkv * d + 2 * own * hkv * d)
print(f"rope_qkv us={us:.1f} GB/s={nbytes / us / 1e3:.0f}")
if len(sys.argv) > 2 and sys.argv[1] == "--check":
    sample = [qo[::97].cpu(), ko[::97].cpu(), kp.cpu(), vp.cpu()]
    if os.path.exists(sys.argv[2]):
        ref = torch.load(sys.argv[2])
        print("bit_identical", all(torch.equal(a, b) for a, b in zip(sample, ref)))
    else:
        torch.save(sample, sys.argv[2])
