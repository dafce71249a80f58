"""Debug: K2 query-encode (tcgen05) vs the mma.sync path on one config; run twice with
STAR_K2_QE=1/0 and --cmp to diff."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17116_b200 import ops  # noqa: E402

lq, tail, hq, hkv, d, lens, splits = 8, 8, 32, 8, 128, [3000, 64], 0
if len(sys.argv) > 2:
    lq = tail = int(sys.argv[2])
    lens = [int(x) for x in sys.argv[3].split(",")]
page = 64
g = torch.Generator().manual_seed(1)
B = len(lens)
pps = (max(lens) + page - 1) // page
kp = torch.randn(B * pps + 5, hkv, page, d, generator=g).to(torch.bfloat16).cuda()
vp = torch.randn(B * pps + 5, hkv, page, d, generator=g).to(torch.bfloat16).cuda()
table = torch.randperm(B * pps + 5, generator=g)[:B * pps].to(torch.int32).view(B, pps).cuda()
q = torch.randn(B, lq, hq, d, generator=g).to(torch.bfloat16).cuda()
kv_len = torch.tensor(lens, dtype=torch.int32).cuda()
out, lse = ops.phase2_partial(q, kp, vp, table, kv_len, max(lens), own_tail=tail, n_splits=splits)
torch.cuda.synchronize()
tag = os.environ.get("STAR_K2_QE", "1")
torch.save((out.cpu(), lse.cpu()), f"/tmp/qe_{tag}.pt")
if sys.argv[1:2] == ["--cmp"]:
    a, la = torch.load("/tmp/qe_1.pt")
    b_, lb = torch.load("/tmp/qe_0.pt")
    for bi in range(B):
        for h in range(0, hq, 4):
            e = (a[bi, :, h] - b_[bi, :, h]).abs().max().item()
            el = (la[bi, :, h] - lb[bi, :, h]).abs().max().item()
            print(f"b={bi} h={h} max|d out|={e:.3e} max|d lse|={el:.3e}")
        rows = (a[bi] - b_[bi]).abs().amax(dim=-1)  # [lq, hq]
        print("rows with err>1e-2 (token, head):", (rows > 1e-2).nonzero().tolist()[:20])
