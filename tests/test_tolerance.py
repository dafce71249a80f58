"""Why the bf16 parity bound is stated the way it is (CPU, no GPU).

Exact (fp64) causal attention with ONLY the softmax weights P rounded to bf16 before P.V —
the single rounding a tensor-core flash attention adds on bf16 inputs with fp32 accumulation —
already exceeds 2e-3 in max-norm per (128-row block, head), while staying under one bf16
rounding unit (2^-8) per block and under 2e-3 per head (Frobenius).  tests/test_fullsize_gpu.py
uses exactly these two bounds for K1."""

import numpy as np
import torch

from oracle import star_oracle as O


def test_bf16_p_quantisation_floor():
    m, d = 1024, 128
    q, k, v = (torch.from_numpy(O.counter_fill(s, m * d).reshape(m, d).astype(np.float32))
               .bfloat16().double() for s in (31, 32, 33))
    s = (q @ k.T) / np.sqrt(d)
    s = s.masked_fill(torch.triu(torch.ones(m, m, dtype=torch.bool), 1), -float("inf"))
    p = torch.exp(s - s.max(1, keepdim=True).values)
    ref = (p @ v) / p.sum(1, keepdim=True)
    pb = p.float().bfloat16().double()
    o = (pb @ v) / pb.sum(1, keepdim=True)
    blk = ((o - ref).abs().view(m // 128, 128, d).amax((1, 2))
           / ref.abs().view(m // 128, 128, d).amax((1, 2)))
    fro = float((o - ref).norm() / ref.norm())
    assert float(blk.max()) > 2e-3          # the per-block 2e-3 is below the floor ...
    assert float(blk.max()) <= 2.0 ** -8     # ... one bf16 unit is not
    assert fro <= 2e-3
