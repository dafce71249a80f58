"""Where the e2e (host-buffer) phase-1 step loses time against the device-resident step.

cfg2 at N = 1, augmented host layout: times pipeline._encode with (a) H2D + D2H, (b) no
H2D (inputs already staged), (c) no D2H, (d) neither (per-part compute structure only),
and (e) the one-launch device step (rope_qkv + K1 over all segments)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_17116_b200 import ops, pipeline  # noqa: E402

L, b, a, hq, hkv, d = 131072, 16384, 16384, 32, 8, 128
dev = torch.device("cuda", 0)
n = L // b
seg, own, pos = [0], [], []
for i in range(n):
    m = b + (a if i else 0)
    seg.append(seg[-1] + m)
    own.append(b)
    pos.append(np.concatenate([np.arange(a), np.arange(i * b, i * b + b)]) if i else np.arange(b))
R = seg[-1]
positions = torch.from_numpy(np.concatenate(pos)).to(dev)
q = ops.prng_fill((R, hq, d), 1, 1, 1.0, torch.bfloat16, dev)
k = ops.prng_fill((R, hkv, d), 2, 1, 1.0, torch.bfloat16, dev)
v = ops.prng_fill((R, hkv, d), 3, 1, 1.0, torch.bfloat16, dev)
hq_, hk_, hv_ = (torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in (q, k, v))
hq_.copy_(q), hk_.copy_(k), hv_.copy_(v)
hout = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
dout = torch.empty_like(q)
pages = L // 128 + 1
kp = torch.zeros((pages, hkv, 128, d), dtype=torch.bfloat16, device=dev)
vp = torch.zeros_like(kp)
table = torch.arange(pages, dtype=torch.int32, device=dev)
plan = pipeline.LayerEncodePlan.create(seg, own, hq, hkv, d, dev)
plan.q.copy_(q), plan.k.copy_(k), plan.v.copy_(v)


def copy_in(i, r0, r1):
    plan.q[r0:r1].copy_(hq_[r0:r1], non_blocking=True)
    plan.k[r0:r1].copy_(hk_[r0:r1], non_blocking=True)
    plan.v[r0:r1].copy_(hv_[r0:r1], non_blocking=True)


def no_copy(i, r0, r1):
    pass


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {
    "h2d+d2h": timed(lambda: pipeline._encode(plan, copy_in, positions, kp, vp, table, hout, 1e4)),
    "no h2d": timed(lambda: pipeline._encode(plan, no_copy, positions, kp, vp, table, hout, 1e4)),
    "no d2h": timed(lambda: pipeline._encode(plan, copy_in, positions, kp, vp, table, dout, 1e4)),
    "neither": timed(lambda: pipeline._encode(plan, no_copy, positions, kp, vp, table, dout, 1e4)),
}
cr = torch.full((R,), -1, dtype=torch.int64)
c0 = 0
for i in range(n):
    cr[seg[i + 1] - own[i]:seg[i + 1]] = torch.arange(c0, c0 + own[i])
    c0 += own[i]
cr = cr.to(dev)
qr, kr = torch.empty_like(q), torch.empty_like(k)


def device_step():
    ops.rope_qkv(q, k, v, positions, 1e4, q_out=qr, k_out=kr, cache_rows=cr, k_pages=kp,
                 v_pages=vp, page_table=table)
    ops.phase1_fwd(qr, kr, v, seg, out=dout)


res["device one-launch"] = timed(device_step)


def device_per_block():
    for i in range(n):
        a0, a1 = seg[i], seg[i + 1]
        ops.rope_qkv(q[a0:a1], k[a0:a1], v[a0:a1], positions[a0:a1], 1e4, q_out=qr[a0:a1],
                     k_out=kr[a0:a1], cache_rows=cr[a0:a1], k_pages=kp, v_pages=vp,
                     page_table=table)
        ops.phase1_fwd(qr[a0:a1], kr[a0:a1], v[a0:a1], [0, a1 - a0], out=dout[a0:a1])


res["device per-block launches"] = timed(device_per_block)
t0 = timed(lambda: hout.copy_(dout, non_blocking=True), 3)
t1 = timed(lambda: plan.q.copy_(hq_, non_blocking=True), 3)
res["d2h 2.0 GB alone"] = t0
res["h2d q 2.0 GB alone"] = t1
print({k: round(x, 2) for k, x in res.items()})
