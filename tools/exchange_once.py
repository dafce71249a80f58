"""A few one-box star_phase2_exchange calls (fused K2 + push + merge) for ncu captures."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17116_b200 import dist as D  # noqa: E402
from paper_2411_17116_b200 import ops  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
dev = torch.device("cuda", 0)
hq, hkv, d, ps = 32, 8, 128, 128
pages = rows // ps
kp = ops.prng_fill((pages, hkv, ps, d), 2, 1, 1.0, torch.bfloat16, dev)
vp = ops.prng_fill((pages, hkv, ps, d), 3, 1, 1.0, torch.bfloat16, dev)
table = torch.arange(pages, dtype=torch.int32, device=dev).view(1, -1)
kv_len = torch.tensor([rows], dtype=torch.int32, device=dev)
q = ops.prng_fill((1, 1, hq, d), 4, 1, 1.0, torch.bfloat16, dev)
ex = D.local_peer_exchanges(1, hq, hkv, d, dev)[0]
ws = ops.Phase2Workspace()
for _ in range(8):
    out, lse = ex.exchange(q, kp, vp, table, kv_len, rows, workspace=ws)
torch.cuda.synchronize()
ref, _ = ops.phase2_partial(q, kp, vp, table, kv_len, rows)
assert torch.equal(out, ref), "one-box exchange must equal plain K2"
print("ok", rows)
