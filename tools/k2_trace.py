"""K2 timeline across CTAs from the tracing library (globaltimer ns; make -C csrc trace).

    python tools/k2_trace.py [--rows 16384] [--batch 1]

Prints, relative to the earliest CTA entry: the spread of CTA entry, first tile landed, main
loop end, split stored, fix-up poll satisfied, and CTA exit — i.e. where the tail of a
short-context decode goes.
"""
import argparse
import ctypes
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
p.add_argument("--rows", type=int, default=16384)
p.add_argument("--batch", type=int, default=1)
p.add_argument("--splits", type=int, default=0)
p.add_argument("--exchange", action="store_true", help="fused star_phase2_exchange (self-loop)")
p.add_argument("--decode", action="store_true", help="fused decode step (star_phase2_decode)")
a = p.parse_args()
dev = torch.device("cuda", 0)
hq, hkv, d, page = 32, 8, 128, 128
pages = -(-a.rows // page) * a.batch
kp = ops.prng_fill((pages, hkv, page, d), 5, 1, 1.0, torch.bfloat16, dev)
vp = ops.prng_fill((pages, hkv, page, d), 6, 1, 1.0, torch.bfloat16, dev)
table = torch.arange(pages, dtype=torch.int32, device=dev).view(a.batch, -1)
q = ops.prng_fill((a.batch, 1, hq, d), 7, 1, 1.0, torch.bfloat16, dev)
kv_len = torch.full((a.batch,), a.rows, dtype=torch.int32, device=dev)
ws = ops.Phase2Workspace()
splits = a.splits or lib.star_phase2_auto_splits(a.batch, hkv, a.rows, page)
ncta = splits * hkv * a.batch
if a.exchange:
    from paper_2411_17116_b200 import dist as D
    ex = D.local_peer_exchanges(1, hq * a.batch, hkv * a.batch, d, dev)[0]
kn = ops.prng_fill((a.batch, hkv, d), 8, 1, 1.0, torch.bfloat16, dev)
vn = ops.prng_fill((a.batch, hkv, d), 9, 1, 1.0, torch.bfloat16, dev)
pos = torch.full((a.batch,), a.rows - 1, dtype=torch.int64, device=dev)
rtab = ops.RopeTable(a.rows - 1, 8, d, 10000.0, dev)
for _ in range(20):
    if a.decode:
        kv_len.fill_(a.rows - 1)
        ops.phase2_decode(q.view(a.batch, hq, d), kn, vn, pos, kp, vp, table, kv_len, a.rows,
                          table=rtab, n_splits=splits, workspace=ws)
    elif a.exchange:
        ex.exchange(q, kp, vp, table, kv_len, a.rows, n_splits=splits, workspace=ws)
    else:
        ops.phase2_partial(q, kp, vp, table, kv_len, a.rows, n_splits=splits, workspace=ws)
torch.cuda.synchronize()
S = 12  # slots per CTA (phase2_mma.cu kK2TrSlots)
N = 2048 * S
buf = (ctypes.c_ulonglong * N)()
lib.star_debug_k2_trace.restype = ctypes.c_int
lib.star_debug_k2_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.star_debug_k2_trace(buf, N)
t = np.frombuffer(buf, dtype=np.uint64).reshape(2048, S)[:ncta].astype(np.int64)
t0 = t[:, 0].min()
names = ["entry", "first tile", "loop done", "stored", "fixup seen", "exit", "xchg seen",
         "xchg arrived", "kv_len read", "loop done g1", "all loops", "staged"]
order = [0, 8, 1, 2, 9, 10, 11, 3, 4, 5, 6, 7]
print(f"rows={a.rows} batch={a.batch} splits={splits} ctas={ncta}")
for j in order:
    nm = names[j]
    col = t[:, j]
    col = col[col > 0] - t0
    if len(col):
        print(f"  {nm:11s} min {col.min()/1e3:7.2f} us  median {np.median(col)/1e3:7.2f}  max {col.max()/1e3:7.2f}")
