"""One causal launch on a 32,768-row block (cfg2's unit, 32 q / 8 kv heads, d 128, bf16) of
either our K1 or cuDNN SDPA, for an ncu side-by-side (tools/gpu/r02f.sh).
Usage: python tools/k1_vs_cudnn.py ours|cudnn [rows] [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_17116_b200 import ops  # noqa: E402

which = sys.argv[1]
m = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
hq, hkv, d = 32, 8, 128
dev = torch.device("cuda", 0)
q = ops.prng_fill((m, hq, d), 31, 1, 1.0, torch.bfloat16, dev)
k = ops.prng_fill((m, hkv, d), 32, 1, 1.0, torch.bfloat16, dev)
v = ops.prng_fill((m, hkv, d), 33, 1, 1.0, torch.bfloat16, dev)
torch.cuda.synchronize()
if which == "ours":
    o = torch.empty_like(q)
    for _ in range(reps):
        ops.phase1_fwd(q, k, v, [0, m], out=o)
else:
    import torch.nn.functional as F
    from torch.nn.attention import SDPBackend, sdpa_kernel

    qt, kt, vt = (x.transpose(0, 1).unsqueeze(0) for x in (q, k, v))
    with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
        for _ in range(reps):
            F.scaled_dot_product_attention(qt, kt, vt, is_causal=True, enable_gqa=True)
torch.cuda.synchronize()
print("done", which, m)
