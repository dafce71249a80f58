"""K2q timeline of CTA 0 (clock64, tracing library: make -C paper_2411_17116_b200/csrc trace).

    python tools/k2q_trace.py [--rows 131072] [--lq 32]

Per tile: softmax warp 0 (S seen, half max, maxima swapped, exps+packs, P handed over) and
the MMA lane (P seen, P.V issued, next S issued), plus steady-state averages."""
import argparse
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

p = argparse.ArgumentParser()
p.add_argument("--rows", type=int, default=131072)
p.add_argument("--lq", type=int, default=32)
a = p.parse_args()
dev = torch.device("cuda", 0)
hq, hkv, d, ps = 32, 8, 128, 128
pages = a.rows // ps
kp = ops.prng_fill((pages, hkv, ps, d), 2, 1, 1.0, torch.bfloat16, dev)
vp = ops.prng_fill((pages, hkv, ps, d), 3, 1, 1.0, torch.bfloat16, dev)
table = torch.arange(pages, dtype=torch.int32, device=dev).view(1, -1)
kv_len = torch.tensor([a.rows], dtype=torch.int32, device=dev)
q = ops.prng_fill((1, a.lq, hq, d), 4, 1, 1.0, torch.bfloat16, dev)
for _ in range(5):
    ops.phase2_partial(q, kp, vp, table, kv_len, a.rows, own_tail=a.lq)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * (256 * 8))()
lib.star_debug_k2q_trace.restype = ctypes.c_int
lib.star_debug_k2q_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.star_debug_k2q_trace(buf, 256 * 8)
t = np.frombuffer(buf, dtype=np.int64).reshape(256, 8).copy()
n = int((t[:, 0] > 0).sum())
t = t[:n]
t0 = t[0, 0]
print("tile: S_seen max swap exps P_out | P_seen PV_issued S_issued   (clk from t0)")
for j in list(range(min(6, n))) + list(range(max(6, n - 3), n)):
    print(f"{j:4d}: " + " ".join(f"{x - t0:8d}" for x in t[j]))
ss = t[4:n - 2]
res = {
    "tiles": n,
    "period_clk": float(np.mean(np.diff(t[4:n - 2, 0]))),
    "ld_max": float(np.mean(ss[:, 1] - ss[:, 0])),
    "swap": float(np.mean(ss[:, 2] - ss[:, 1])),
    "exps_pack": float(np.mean(ss[:, 3] - ss[:, 2])),
    "store_handoff": float(np.mean(ss[:, 4] - ss[:, 3])),
    "p_to_mma_seen": float(np.mean(ss[:, 5] - ss[:, 4])),
    "pv_issue": float(np.mean(ss[:, 6] - ss[:, 5])),
    "s_issue": float(np.mean(ss[:, 7] - ss[:, 6])),
    "p_out_to_next_s_seen": float(np.mean(t[5:n - 1, 0] - t[4:n - 2, 4])),
}
print(json.dumps(res))
