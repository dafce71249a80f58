"""K1 timeline of CTA 0 (the heaviest q tile of segment 0) from the tracing library.

Build: make -C paper_2411_17116_b200/csrc trace.  Run on the GPU box:
    python tools/k1_trace.py [env STAR_K1_*]
Prints per-tile softmax phases (S ready -> max -> turn -> exps -> P handed over) and the
MMA warp's view (P seen -> PV + next S issued), in SM clocks, plus steady-state averages.
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_17116_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.join(ROOT, "paper_2411_17116_b200", "libstar_attn_trace.so")
lib = _lib.load()
from paper_2411_17116_b200 import ops  # noqa: E402

L, b, hq, hkv, d = 131072, 16384, 32, 8, 128
dev = torch.device("cuda", 0)
n = L // b
seg = [0]
for i in range(n):
    seg.append(seg[-1] + b + (b if i else 0))
R = seg[-1]
q = ops.prng_fill((R, hq, d), 1, 1, 1.0, torch.bfloat16, dev)
k = ops.prng_fill((R, hkv, d), 2, 1, 1.0, torch.bfloat16, dev)
v = ops.prng_fill((R, hkv, d), 3, 1, 1.0, torch.bfloat16, dev)
out = torch.empty_like(q)
for _ in range(3):
    ops.phase1_fwd(q, k, v, seg, out=out)
torch.cuda.synchronize()
N = 2 * 256 * 5 + 256 * 2 * 2 + 2 * 256 * 4 * 2
buf = (ctypes.c_longlong * N)()
lib.star_debug_k1_trace.restype = ctypes.c_int
assert lib.star_debug_k1_trace(buf, N) == N
a = np.frombuffer(buf, dtype=np.int64).copy()
sm = a[:2 * 256 * 5].reshape(2, 256, 5)
mm = a[2 * 256 * 5:2 * 256 * 5 + 256 * 4].reshape(256, 2, 2)
wq = a[2 * 256 * 5 + 256 * 4:].reshape(2, 256, 4, 2)  # [head][tile][quarter][S seen, P out]
ntiles = b // 128
t0 = min(sm[0, 0, 0], sm[1, 0, 0])
print("tile  head: S_ready max_done turn exps_done P_out | mma: P_seen issued   (clk from t0)")
for j in list(range(0, 6)) + list(range(60, 64)) + list(range(ntiles - 3, ntiles)):
    for i in range(2):
        e = sm[i, j] - t0
        m = mm[j, i] - t0
        print(f"{j:4d} {i:2d}: " + " ".join(f"{x:8d}" for x in e) + " | " + " ".join(f"{x:8d}" for x in m))
rng = slice(8, ntiles - 4)
per = np.diff(sm[0, :, 0])[rng].mean()
stat = {
    "period_clk": float(per),
    "max_pass": float((sm[:, rng, 1] - sm[:, rng, 0]).mean()),
    "turn_wait": float((sm[:, rng, 2] - sm[:, rng, 1]).mean()),
    "exps": float((sm[:, rng, 3] - sm[:, rng, 2]).mean()),
    "handoff": float((sm[:, rng, 4] - sm[:, rng, 3]).mean()),
    "p_to_next_s": float((sm[:, 9:ntiles - 3, 0] - sm[:, 8:ntiles - 4, 4]).mean()),
    "mma_issue": float((mm[rng, :, 1] - mm[rng, :, 0]).mean()),
    "p_out_to_mma_seen": float((mm[rng, :, 0] - sm[:, rng, 4].T).mean()),
    "quarter_s_seen_minus_min": [float(x) for x in (wq[:, rng, :, 0] - wq[:, rng, :, 0].min(axis=2, keepdims=True)).mean(axis=(0, 1))],
    "quarter_p_out_minus_min": [float(x) for x in (wq[:, rng, :, 1] - wq[:, rng, :, 1].min(axis=2, keepdims=True)).mean(axis=(0, 1))],
    "mma_seen_minus_last_quarter_p": float((mm[rng, :, 0] - wq[:, rng, :, 1].max(axis=2).T).mean()),
    "issued_to_next_s": float((sm[:, 9:ntiles - 3, 0].T - mm[8:ntiles - 4, :, 1]).mean()),
    "knobs": {k_: v_ for k_, v_ in os.environ.items() if k_.startswith("STAR_K1_")},
}
print(json.dumps(stat))
