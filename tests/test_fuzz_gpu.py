"""Seeded randomized parity sweep of the compute entry points against the fp64 oracle.

Each case draws its own shape from a fixed seed (so a failure names a reproducible case):
  * K1 (`phase1_fwd`, tcgen05 for bf16, the CUDA-core check kernel for fp32): 1-4 causal
    segments of 1-900 rows (ragged against the 128-row tiles), GQA ratio 1-8 (odd ratios run
    one q head per CTA), head_dim 64/128, input amplitude 0.25-4 (flat to sharp softmax);
  * K2 / K2q (`phase2_partial`): batch 1-5 of 1-6000 cached rows over a permuted page table
    (page 64 or 128), 1-32 query rows with or without the own-tail mask, automatic or explicit
    1-8 split counts, fp32 and bf16.
Tolerances against the oracle on the same rounded inputs: fp32 rel 1e-5; K1 bf16
(P rounded to bf16 before P.V) Frobenius-relative <= 2e-3 per (segment, head) and max-norm
<= 2^-8 per (128-row block, head); K2 / K2q bf16 (P carried as a hi/lo pair) normwise <= 2e-3
per (sequence, head); lse abs 2e-3.
"""

import numpy as np
import pytest
import torch

from oracle import star_oracle as O

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-3
GEOMS = [(4, 4), (8, 2), (8, 1), (12, 4), (16, 4), (32, 8), (64, 8), (10, 2)]


@pytest.fixture(scope="module")
def ops():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2411_17116_b200 import ops as _ops
    return _ops


def _normwise(a, ref):
    return float(np.max(np.abs(a - ref)) / max(np.max(np.abs(ref)), 1e-30))


def _k1_bf16_errors(got, ref):
    """(Frobenius-relative error of the segment, worst max-norm error of its 128-row blocks)."""
    fro = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
    blk = max(_normwise(got[r:r + 128], ref[r:r + 128]) for r in range(0, len(ref), 128))
    return fro, blk


@pytest.mark.parametrize("case", range(32))
def test_phase1_random_shapes(ops, case):
    rng = np.random.default_rng(1000 + case)
    hq, hkv = GEOMS[rng.integers(len(GEOMS))]
    d = int(rng.choice([64, 128]))
    dtype = torch.float32 if case % 4 == 3 else torch.bfloat16
    lens = [int(x) for x in rng.integers(1, 901, size=int(rng.integers(1, 5)))]
    amp = float(rng.choice([0.25, 1.0, 2.0, 4.0]))
    if dtype == torch.float32:
        # the fp32 check mode's 1e-5 holds for O(1) logits: an fp32 score of
        # magnitude |s| carries ~|s| * 2^-24 * sqrt(d) absolute error into exp(s) (the
        # reference computes its scores in fp32 too), so keep |s| = O(1) here
        amp = min(amp, 1.0)
    rows = sum(lens)
    gen = torch.Generator().manual_seed(case)
    q = (amp * torch.randn(rows, hq, d, generator=gen)).to(dtype)
    k = (amp * torch.randn(rows, hkv, d, generator=gen)).to(dtype)
    v = torch.randn(rows, hkv, d, generator=gen).to(dtype)
    starts = np.concatenate([[0], np.cumsum(lens)]).tolist()
    out, lse = ops.phase1_fwd(q.cuda(), k.cuda(), v.cuda(), starts, want_lse=True,
                              out_dtype=torch.float32)
    torch.cuda.synchronize()
    got, got_lse = out.cpu().numpy(), lse.cpu().numpy()
    qn, kn, vn = (t.float().numpy().astype(np.float64) for t in (q, k, v))
    G = hq // hkv
    for a, b in zip(starts[:-1], starts[1:]):
        for h in range(hq):
            ref, ref_lse = O.causal_attention_lse(qn[a:b, h], kn[a:b, h // G], vn[a:b, h // G])
            if dtype == torch.float32:
                np.testing.assert_allclose(got[a:b, h], ref, rtol=1e-5, atol=1e-6)
                np.testing.assert_allclose(got_lse[h, a:b], ref_lse, rtol=1e-6, atol=1e-5)
            else:
                fro, blk = _k1_bf16_errors(got[a:b, h], ref)
                assert fro <= BF16_TOL and blk <= 2.0 ** -8, (case, hq, hkv, d, lens, amp, h, a, fro, blk)
                assert np.abs(got_lse[h, a:b] - ref_lse).max() <= BF16_TOL, (case, h, a)


@pytest.mark.parametrize("case", range(40))
def test_phase2_random_shapes(ops, case):
    rng = np.random.default_rng(2000 + case)
    hq, hkv = GEOMS[rng.integers(len(GEOMS))]
    d = int(rng.choice([64, 128]))
    dtype = torch.float32 if case % 4 == 3 else torch.bfloat16
    lq = int(rng.choice([1, 1, 2, 5, 16, 32]))
    B = int(rng.integers(1, 6))
    own_tail = lq if rng.random() < 0.4 else 0
    lens = [int(x) for x in rng.integers(max(lq, 1), 6001, size=B)]
    page = int(rng.choice([64, 128]))
    splits = 0 if rng.random() < 0.5 else int(rng.integers(1, 9))
    if splits > 1 and splits * (hq // hkv) * lq * 4 + (hq // hkv) * lq * 4 + 16 > 6 * 16384:
        splits = 0  # the in-kernel fix-up buffer bounds splits x query rows (ConfigError)
    pps = (max(lens) + page - 1) // page
    n_pages = B * pps + 3
    kpool = torch.zeros((n_pages, hkv, page, d), dtype=dtype, device="cuda")
    vpool = torch.zeros_like(kpool)
    table = torch.from_numpy(rng.permutation(n_pages)[:B * pps].astype(np.int32).reshape(B, pps)).cuda()
    gen = torch.Generator().manual_seed(case)
    q = torch.randn(B, lq, hq, d, generator=gen).to(dtype)
    ks, vs = [], []
    for b, L in enumerate(lens):
        k = (1.5 * torch.randn(L, hkv, d, generator=gen)).to(dtype)
        v = torch.randn(L, hkv, d, generator=gen).to(dtype)
        ops.kv_write(k.cuda(), v.cuda(), kpool, vpool, table[b].contiguous(), 0)
        ks.append(k)
        vs.append(v)
    kv_len = torch.tensor(lens, dtype=torch.int32).cuda()
    out, lse = ops.phase2_partial(q.cuda(), kpool, vpool, table, kv_len, max(lens),
                                  own_tail=own_tail, n_splits=splits)
    torch.cuda.synchronize()
    G = hq // hkv
    got, got_lse = out.cpu().numpy(), lse.cpu().numpy()
    for b, L in enumerate(lens):
        keep = "full"
        if own_tail:
            keep = np.ones((lq, L), dtype=bool)
            keep[:, L - own_tail:] = O.causal_keep(lq, own_tail)
        kk_all = ks[b].float().numpy().astype(np.float64)
        vv_all = vs[b].float().numpy().astype(np.float64)
        for h in range(hq):
            qq = q[b, :, h].float().numpy().astype(np.float64)
            ref, ref_lse = O.partial_attention(qq, kk_all[:, h // G], vv_all[:, h // G], keep)
            if dtype == torch.float32:
                np.testing.assert_allclose(got[b, :, h], ref, rtol=1e-5, atol=1e-6)
                np.testing.assert_allclose(got_lse[b, :, h], ref_lse, rtol=1e-6, atol=1e-5)
            else:
                err = _normwise(got[b, :, h], ref)
                assert err <= BF16_TOL, (case, hq, hkv, d, lq, lens, own_tail, splits, b, h, err)
                assert np.abs(got_lse[b, :, h] - ref_lse).max() <= BF16_TOL, (case, b, h)


@pytest.mark.parametrize("case", range(12))
def test_fused_decode_random_chains(ops, case):
    """A random multi-token decode chain through star_phase2_decode + star_decode_advance is
    BIT-IDENTICAL, token by token, to star_kv_append + star_phase2_partial (pages, out, lse):
    batch 1-4, G 1-8, d 64/128, ragged starting lengths (empty caches, page and tile edges),
    auto or explicit split counts, 1-6 tokens."""
    rng = np.random.default_rng(3000 + case)
    hq, hkv = [(32, 8), (8, 2), (8, 8), (16, 2), (64, 8)][rng.integers(5)]
    d = int(rng.choice([64, 128]))
    B = int(rng.integers(1, 5))
    page = 128
    edges = [0, 63, 64, 127, 128, 4095, 4096]
    starts = [int(rng.choice(edges)) if rng.random() < 0.5 else int(rng.integers(0, 6000))
              for _ in range(B)]
    n_tok = int(rng.integers(1, 7))
    splits = 0 if rng.random() < 0.6 else int(rng.integers(1, 9))
    maxk = max(starts) + n_tok + 64
    pps = -(-maxk // page)
    gen = torch.Generator().manual_seed(case)
    dev = torch.device("cuda")
    table = torch.from_numpy(rng.permutation(B * pps).astype(np.int32).reshape(B, pps)).cuda()
    kp = ops.prng_fill((B * pps, hkv, page, d), 10 + case, 1, 1.0, torch.bfloat16, dev)
    vp = ops.prng_fill((B * pps, hkv, page, d), 50 + case, 1, 1.0, torch.bfloat16, dev)
    kp_r, vp_r = kp.clone(), vp.clone()
    kl = torch.tensor(starts, dtype=torch.int32).cuda()
    kl_r = kl.clone()
    pos = torch.tensor([s + 3 for s in starts], dtype=torch.int64).cuda()
    pos_r = pos.clone()
    for t in range(n_tok):
        q = torch.randn(B, hq, d, generator=gen).bfloat16().cuda()
        k = torch.randn(B, hkv, d, generator=gen).bfloat16().cuda()
        v = torch.randn(B, hkv, d, generator=gen).bfloat16().cuda()
        qr = ops.kv_append(q, k, v, pos_r, kl_r, kp_r, vp_r, table)
        o_r, l_r = ops.phase2_partial(qr.view(B, 1, hq, d), kp_r, vp_r, table, kl_r, maxk,
                                      n_splits=splits)
        pos_r += 1
        o, l = ops.phase2_decode(q, k, v, pos, kp, vp, table, kl, maxk, n_splits=splits)
        ops.decode_advance(kl, pos)
        torch.cuda.synchronize()
        assert torch.equal(o, o_r) and torch.equal(l, l_r), (case, t)
        assert torch.equal(kl, kl_r) and torch.equal(pos, pos_r), (case, t)
    assert torch.equal(kp, kp_r) and torch.equal(vp, vp_r), case
