"""K2 (bf16 split-KV decode) normwise error vs the fp64 oracle across attention sharpness —
used to pick the P.V precision knob (STAR_K2_PLO).  Prints the max normwise error per case."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import star_oracle as O  # noqa: E402  (test infrastructure: the checker)
from paper_2411_17116_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
d, hq, hkv, page = 128, 32, 8, 128
for rows in (300, 4096, 65536):
    for qscale in (0.25, 1.0, 4.0, 16.0):
        pages = -(-rows // page)
        kp = ops.prng_fill((pages, hkv, page, d), 5, 1, 1.0, torch.bfloat16, dev)
        vp = ops.prng_fill((pages, hkv, page, d), 6, 1, 1.0, torch.bfloat16, dev)
        table = torch.arange(pages, dtype=torch.int32, device=dev).view(1, -1)
        q = ops.prng_fill((1, 1, hq, d), 7, 1, qscale, torch.bfloat16, dev)
        kv_len = torch.tensor([rows], dtype=torch.int32, device=dev)
        out, lse = ops.phase2_partial(q, kp, vp, table, kv_len, rows)
        torch.cuda.synchronize()
        kd = kp.permute(1, 0, 2, 3).reshape(hkv, -1, d)[:, :rows].float().cpu().numpy().astype(np.float64)
        vd = vp.permute(1, 0, 2, 3).reshape(hkv, -1, d)[:, :rows].float().cpu().numpy().astype(np.float64)
        worst = wl = 0.0
        for h in range(0, hq, 3):
            qq = q[0, :, h].float().cpu().numpy().astype(np.float64)
            ro, rl = O.partial_attention(qq, kd[h // 4], vd[h // 4])
            worst = max(worst, np.abs(out[0, 0, h].cpu().numpy() - ro[0]).max() / np.abs(ro[0]).max())
            wl = max(wl, abs(float(lse[0, 0, h]) - float(rl[0])))
        print(f"PLO={os.environ.get('STAR_K2_PLO', '1')} rows={rows} qscale={qscale}: normwise {worst:.2e}  lse {wl:.2e}")
