"""K1 accuracy on one 32K-row causal block (cfg2's unit) against the fp32 CUDA-core check
kernel on the same bf16 inputs: worst per-head Frobenius and per-(128-row block, head)
max-norm error, fp32 output.  Prints one JSON line (knobs from STAR_K1_* env)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17116_b200 import ops  # noqa: E402

m, hq, hkv, d = int(sys.argv[1]) if len(sys.argv) > 1 else 32768, 32, 8, 128
dev = torch.device("cuda", 0)
q = ops.prng_fill((m, hq, d), 31, 1, 1.0, torch.bfloat16, dev)
k = ops.prng_fill((m, hkv, d), 32, 1, 1.0, torch.bfloat16, dev)
v = ops.prng_fill((m, hkv, d), 33, 1, 1.0, torch.bfloat16, dev)
o, lse = ops.phase1_fwd(q, k, v, [0, m], want_lse=True, out_dtype=torch.float32)
r, rl = ops.phase1_fwd_check(q, k, v, [0, m])
nb = m // 128
blk = ((o - r).abs().view(nb, 128, hq, d).amax(dim=(1, 3)) / r.abs().view(nb, 128, hq, d).amax(dim=(1, 3)))
fro = ((o - r).pow(2).sum(dim=(0, 2)).sqrt() / r.pow(2).sum(dim=(0, 2)).sqrt()).max()
print(json.dumps({"knobs": {k_: v_ for k_, v_ in os.environ.items() if k_.startswith("STAR_K1_")},
                  "block_max": float(blk.max()), "block_p999": float(blk.flatten().quantile(0.999)),
                  "fro_max_head": float(fro), "lse_max_abs": float((lse - rl).abs().max())}))
