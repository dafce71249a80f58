"""Kernel parity on the B200: every C-ABI compute entry point against the CPU oracle.

Tolerances (written here, per BASELINE.json north_star):
  * fp32 check mode: rel 1e-5 (elementwise, atol 1e-6) — SPEC.md:181.
  * bf16 inputs with fp32 accumulation: normwise max|d| / max|ref| <= 2e-3 per head,
    compared against the oracle run on the SAME bf16-rounded inputs; lse abs <= 2e-3.
  * integer / layout / PRNG items: bit-exact.
"""

import numpy as np
import pytest
import torch

from oracle import star_oracle as O

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-3
# a bf16 OUTPUT adds up to half an ulp (2^-9 relative) of rounding on top of the kernel's
# arithmetic error; bf16-output comparisons allow for it explicitly.
BF16_OUT_TOL = BF16_TOL + 2.0 ** -9


@pytest.fixture(scope="module")
def ops():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2411_17116_b200 import ops as _ops
    return _ops


def t2n(t):
    return t.detach().float().cpu().numpy()


def normwise(a, ref):
    return float(np.max(np.abs(a - ref)) / max(np.max(np.abs(ref)), 1e-30))


# --------------------------------------------------------------------------- UMMA descriptors
@pytest.mark.parametrize("a_tmem", [False, True])
@pytest.mark.parametrize("mn", [False, True])
@pytest.mark.parametrize("K", [64, 128, 256])
def test_umma_descriptor_gemm(ops, mn, K, a_tmem):
    g = torch.Generator(device="cpu").manual_seed(K + mn)
    a = torch.randn(128, K, generator=g).to(torch.bfloat16).cuda()
    b = torch.randn(128, K, generator=g).to(torch.bfloat16).cuda()
    ref = a.float() @ b.float().T
    bb = b.T.contiguous() if mn else b
    c = ops.debug_umma_gemm(a, bb, b_mn_major=mn, a_tmem=a_tmem)
    torch.cuda.synchronize()
    assert torch.allclose(c, ref, rtol=1e-4, atol=1e-3), float((c - ref).abs().max())


# --------------------------------------------------------------------------- PRNG
@pytest.mark.parametrize("seed", [0, 7, 0xA17C4B10C4ED5EED])
def test_prng_fill_bit_exact(ops, seed):
    n = 100_003
    got = ops.prng_fill((n,), seed, first=1, scale=0.5, dtype=torch.float32)
    ref = O.counter_fill(seed, n, 0.5).astype(np.float32)
    np.testing.assert_array_equal(t2n(got), ref)
    got = ops.prng_fill((n,), seed, first=1, scale=0.5, dtype=torch.bfloat16)
    ref_b = torch.from_numpy(ref).to(torch.bfloat16)
    assert torch.equal(got.cpu(), ref_b)
    # random access: draws 1001.. of the stream
    got = ops.prng_fill((50,), seed, first=1001, scale=0.5)
    np.testing.assert_array_equal(t2n(got), O.counter_fill(seed, 1050, 0.5)[1000:].astype(np.float32))


# --------------------------------------------------------------------------- RoPE
def test_rope_matches_reference_goldens(ops, golden_dir):
    g = np.load(f"{golden_dir}/rope.npz")
    for n in "ab":  # fp32 cases (the fp64 case has no fp64 device path)
        x, pos, y = g[f"{n}_x"], g[f"{n}_pos"], g[f"{n}_y"]
        xt = torch.from_numpy(x).cuda().view(x.shape[0], 1, x.shape[1])
        out = ops.rope(xt, torch.from_numpy(pos).cuda(), float(g[f"{n}_theta"]))
        np.testing.assert_allclose(t2n(out).reshape(y.shape), y, rtol=1e-6, atol=1e-6)


def test_rope_multihead_bf16(ops):
    rng = np.random.default_rng(1)
    rows, heads, d = 77, 5, 128
    x = rng.standard_normal((rows, heads, d)).astype(np.float32)
    pos = rng.integers(0, 1 << 20, rows)
    xb = torch.from_numpy(x).to(torch.bfloat16)
    out = ops.rope(xb.cuda(), torch.from_numpy(pos).cuda())
    xr = xb.float().numpy()
    for h in range(heads):
        ref = O.rope(xr[:, h].astype(np.float64), pos)
        np.testing.assert_allclose(t2n(out)[:, h], ref, rtol=1e-2, atol=1e-2)


# --------------------------------------------------------------------------- dense attention (fp32)
@pytest.mark.parametrize("case", ["c0", "c1", "c2", "c3"])
def test_dense_attention_fp32_goldens(ops, golden_dir, case):
    g = np.load(f"{golden_dir}/attention.npz")
    q, k, v, off = g[f"{case}_q"], g[f"{case}_k"], g[f"{case}_v"], int(g[f"{case}_off"])
    c = lambda a: torch.from_numpy(a).cuda().unsqueeze(1)
    out, lse = ops.attention_dense(c(q), c(k), c(v), q_offset=off, mask="causal")
    np.testing.assert_allclose(t2n(out)[:, 0], g[f"{case}_out"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(t2n(lse)[0], g[f"{case}_pc_lse"], rtol=1e-6, atol=1e-6)
    out, lse = ops.attention_dense(c(q), c(k), c(v), mask="full")
    np.testing.assert_allclose(t2n(out)[:, 0], g[f"{case}_pf_out"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(t2n(lse)[0], g[f"{case}_pf_lse"], rtol=1e-6, atol=1e-6)


# --------------------------------------------------------------------------- phase 1
def _segments_inputs(seg_lens, hq, hkv, d, dtype, seed):
    rows = sum(seg_lens)
    q = torch.from_numpy(O.counter_fill(seed ^ 1, rows * hq * d).astype(np.float32)).view(rows, hq, d)
    k = torch.from_numpy(O.counter_fill(seed ^ 2, rows * hkv * d).astype(np.float32)).view(rows, hkv, d)
    v = torch.from_numpy(O.counter_fill(seed ^ 3, rows * hkv * d).astype(np.float32)).view(rows, hkv, d)
    q, k, v = (t.to(dtype) for t in (q, k, v))
    starts = np.concatenate([[0], np.cumsum(seg_lens)]).tolist()
    return q, k, v, starts


def _oracle_segments(q, k, v, starts, hq, hkv):
    qn, kn, vn = (t.float().numpy().astype(np.float64) for t in (q, k, v))
    G = hq // hkv
    outs, lses = np.zeros_like(qn), np.zeros((hq, qn.shape[0]))
    for a, b in zip(starts[:-1], starts[1:]):
        for h in range(hq):
            o, l = O.causal_attention_lse(qn[a:b, h], kn[a:b, h // G], vn[a:b, h // G])
            outs[a:b, h], lses[h, a:b] = o, l
    return outs, lses


@pytest.mark.parametrize("d,hq,hkv,seg_lens", [
    (128, 8, 2, [128 * 3 + 17, 256]),     # GQA G=4 -> two q heads per CTA, ragged segment
    (128, 4, 4, [300, 129]),              # MHA (one q head per CTA)
    (64, 4, 2, [200, 384, 1]),            # head_dim 64, a 1-row segment
    (128, 32, 8, [1024, 2048]),           # Llama-3.1-8B head geometry, anchor+own block shape
    (128, 64, 8, [700, 300]),             # Llama-3.1-70B heads: 4 head pairs, 4-CTA multicast
])
def test_phase1_tensor_core_bf16(ops, d, hq, hkv, seg_lens):
    q, k, v, starts = _segments_inputs(seg_lens, hq, hkv, d, torch.bfloat16, seed=d + hq)
    ref, ref_lse = _oracle_segments(q, k, v, starts, hq, hkv)
    for out_dtype, tol in ((torch.float32, BF16_TOL), (torch.bfloat16, BF16_OUT_TOL)):
        out, lse = ops.phase1_fwd(q.cuda(), k.cuda(), v.cuda(), starts, want_lse=True,
                                  out_dtype=out_dtype)
        torch.cuda.synchronize()
        got = t2n(out)
        for h in range(hq):
            for a, b in zip(starts[:-1], starts[1:]):
                err = normwise(got[a:b, h], ref[a:b, h])
                assert err <= tol, (out_dtype, h, a, b, err)
        np.testing.assert_allclose(t2n(lse), ref_lse, atol=BF16_TOL, rtol=0)


@pytest.mark.parametrize("knob,value", [("STAR_K1_SM", "1"), ("STAR_K1_SM", "2"),
                                        ("STAR_K1_SM", "3"), ("STAR_K1_SM", "4"),
                                        ("STAR_K1_SM", "5"), ("STAR_K1_SEQ", "1"),
                                        ("STAR_K1_SEQ", "2"), ("STAR_K1_MC", "0")])
@pytest.mark.parametrize("d,hq,hkv,seg_lens", [(128, 8, 2, [128 * 3 + 17, 256]),
                                               (128, 16, 2, [300, 129]),
                                               (64, 4, 2, [200, 384, 1])])
def test_phase1_measurement_knobs(ops, monkeypatch, knob, value, d, hq, hkv, seg_lens):
    """Every K1 form the measurement knobs select (the round-1 kernel, no FMA exp2,
    per-MMA elect, other exp2 shares, the MUFU ping-pong, no K/V multicast) is checked against
    the fp64 oracle like the default form."""
    monkeypatch.setenv(knob, value)  # read by the launcher at every call
    q, k, v, starts = _segments_inputs(seg_lens, hq, hkv, d, torch.bfloat16, seed=d + hq + 7)
    ref, ref_lse = _oracle_segments(q, k, v, starts, hq, hkv)
    out, lse = ops.phase1_fwd(q.cuda(), k.cuda(), v.cuda(), starts, want_lse=True,
                              out_dtype=torch.float32)
    torch.cuda.synchronize()
    got = t2n(out)
    for h in range(hq):
        for a, b in zip(starts[:-1], starts[1:]):
            err = normwise(got[a:b, h], ref[a:b, h])
            assert err <= BF16_TOL, (knob, value, h, a, b, err)
    np.testing.assert_allclose(t2n(lse), ref_lse, atol=BF16_TOL, rtol=0)


@pytest.mark.parametrize("d,hq,hkv,seg_lens", [(64, 4, 4, [100, 64, 33]), (16, 2, 1, [40, 7])])
def test_phase1_fp32_check_mode(ops, d, hq, hkv, seg_lens):
    q, k, v, starts = _segments_inputs(seg_lens, hq, hkv, d, torch.float32, seed=5)
    out, lse = ops.phase1_fwd(q.cuda(), k.cuda(), v.cuda(), starts, want_lse=True)
    ref, ref_lse = _oracle_segments(q, k, v, starts, hq, hkv)
    np.testing.assert_allclose(t2n(out), ref, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(t2n(lse), ref_lse, rtol=1e-6, atol=1e-5)


# --------------------------------------------------------------------------- paged cache + phase 2
def _paged(k, v, page_size, rng):
    """Scatter dense [rows, hkv, d] into a shuffled page pool; returns pools and table."""
    rows, hkv, d = k.shape
    n_pages = (rows + page_size - 1) // page_size
    perm = rng.permutation(n_pages + 3)[:n_pages].astype(np.int32)
    kp = torch.zeros((n_pages + 3, hkv, page_size, d), dtype=k.dtype, device="cuda")
    vp = torch.zeros_like(kp)
    table = torch.from_numpy(perm).cuda()
    return kp, vp, table


def test_kv_write_read_roundtrip(ops):
    rng = np.random.default_rng(3)
    for dtype in (torch.float32, torch.bfloat16):
        k = torch.randn(300, 3, 64).to(dtype).cuda()
        v = torch.randn(300, 3, 64).to(dtype).cuda()
        kp, vp, table = _paged(k, v, 64, rng)
        ops.kv_write(k[:100], v[:100], kp, vp, table, 0)
        ops.kv_write(k[100:], v[100:], kp, vp, table, 100)  # append crossing page boundaries
        k2, v2 = ops.kv_read(kp, vp, table, 0, 300)
        assert torch.equal(k2, k) and torch.equal(v2, v)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("lq,own_tail,hq,hkv,d,lens,splits", [
    (1, 0, 4, 1, 128, [5000], 0),
    (1, 0, 32, 8, 128, [4096, 1, 777], 0),
    (3, 3, 4, 2, 64, [400, 3], 4),
    (5, 0, 8, 8, 64, [1000, 2000], 7),
    (32, 32, 4, 4, 64, [1024 + 32], 0),
    # > 64 query rows per kv head (32-token query encode at Llama-8B heads): two 64-row
    # blocks along grid.y; and 80 rows (a partial second block)
    (32, 32, 32, 8, 128, [5000 + 32, 800], 0),
    (20, 20, 16, 4, 64, [3000], 3),
    # bf16 d=128, 16 < G*l_q <= 128: the tcgen05 query-encode kernel (packed M=128 tile)
    (8, 8, 32, 8, 128, [3000, 64], 0),
    (17, 0, 32, 8, 128, [4000], 5),
    (5, 5, 16, 4, 128, [700], 0),
    (32, 32, 32, 8, 128, [130], 2),
    # K2q with G = 1 (no GQA: 40 tokens x 1 head per tile) and G = 8 (70B heads: 16 x 8)
    (40, 40, 8, 8, 128, [1500], 0),
    (16, 16, 64, 8, 128, [2500], 0),
    # batch 10 x 8 kv heads = 80 groups: one split each, K2q without the fold
    (32, 32, 32, 8, 128, [300 + 97 * i for i in range(10)], 0),
    # G*l_q = 160 > 128: mma.sync row blocks (64 + 64 + 32 rows) at d = 128
    (40, 40, 32, 8, 128, [2000], 0),
    # 19 x 8 = 152 (sequence, kv head) groups >= the SM count: the arrival-counter split
    # fix-up (fewer groups use the word fix-up, where split 0 polls the others' words)
    (1, 0, 8, 8, 64, [300 + 37 * i for i in range(19)], 2),
])
def test_phase2_partial_paged(ops, dtype, lq, own_tail, hq, hkv, d, lens, splits):
    rng = np.random.default_rng(lq * 31 + hq)
    B = len(lens)
    page_size = 64
    pps = (max(lens) + page_size - 1) // page_size
    pools = torch.zeros((B * pps + 5, hkv, page_size, d), dtype=dtype, device="cuda")
    kpool, vpool = pools.clone(), pools.clone()
    table = torch.from_numpy(rng.permutation(B * pps + 5)[:B * pps].astype(np.int32).reshape(B, pps)).cuda()
    q = torch.randn(B, lq, hq, d).to(dtype)
    ks, vs = [], []
    for b, L in enumerate(lens):
        k = torch.randn(L, hkv, d).to(dtype)
        v = torch.randn(L, hkv, d).to(dtype)
        ops.kv_write(k.cuda(), v.cuda(), kpool, vpool, table[b].contiguous(), 0)
        ks.append(k), vs.append(v)
    kv_len = torch.tensor(lens, dtype=torch.int32).cuda()
    out, lse = ops.phase2_partial(q.cuda(), kpool, vpool, table, kv_len, max(lens), own_tail=own_tail,
                                  n_splits=splits)
    torch.cuda.synchronize()
    G = hq // hkv
    got, got_lse = t2n(out), t2n(lse)
    for b, L in enumerate(lens):
        for h in range(hq):
            qq = q[b, :, h].float().numpy().astype(np.float64)
            kk = ks[b][:, h // G].float().numpy().astype(np.float64)
            vv = vs[b][:, h // G].float().numpy().astype(np.float64)
            if own_tail:
                keep = np.ones((lq, L), dtype=bool)
                keep[:, L - own_tail:] = O.causal_keep(lq, own_tail)
            else:
                keep = "full"
            o, l = O.partial_attention(qq, kk, vv, keep)
            if dtype == torch.float32:
                np.testing.assert_allclose(got[b, :, h], o, rtol=1e-5, atol=1e-6)
                np.testing.assert_allclose(got_lse[b, :, h], l, rtol=1e-6, atol=1e-5)
            else:
                assert normwise(got[b, :, h], o) <= BF16_TOL
                np.testing.assert_allclose(got_lse[b, :, h], l, atol=BF16_TOL)


def _rising(n, heads, d, amp, gen, direction=1.0):
    """Rows whose scores against _rising queries grow ~linearly with the row index: key j
    carries amp * j / n along a shared unit direction (plus noise), so every later 128-key
    tile's max exceeds the running max by >> 2^8 (the lazy rescale fires on every tile)."""
    e = torch.ones(d) / d ** 0.5
    ramp = torch.arange(n, dtype=torch.float32).view(n, 1, 1) / n
    return (direction * amp * ramp * e + 0.5 * torch.randn(n, heads, d, generator=gen)).bfloat16()


def _sharp_queries(n, heads, d, gen):
    e = torch.ones(d) / d ** 0.5
    return (3.0 * d ** 0.5 * e + 0.5 * torch.randn(n, heads, d, generator=gen)).bfloat16()


@pytest.mark.parametrize("direction", [1.0, -1.0])
def test_sharp_scores_rescale_paths(ops, direction):
    """Scores spanning ~170 log2 units across the keys, rising (every tile raises the running
    max by >> 2^8: the lazy O / l rescale runs on every tile, and the split partials' lse differ
    by ~100) or falling (the first tile holds the max: no rescale): K1 over two ragged causal
    segments, K2 decode and K2q query encode over a paged cache, each against the fp64 oracle on
    the same bf16 inputs."""
    gen = torch.Generator().manual_seed(11)
    d, hq, hkv, G = 128, 8, 2, 4
    amp = 40.0  # score(q, k_j) ~ 3 * amp * j / n = 120 nats (173 log2) over a segment
    # ---- K1: two causal segments
    seg_lens = [1024 + 300, 700]
    starts = np.concatenate([[0], np.cumsum(seg_lens)]).tolist()
    q = _sharp_queries(sum(seg_lens), hq, d, gen)
    k = torch.cat([_rising(n, hkv, d, amp, gen, direction) for n in seg_lens])
    v = torch.randn(sum(seg_lens), hkv, d, generator=gen).bfloat16()
    out, lse = ops.phase1_fwd(q.cuda(), k.cuda(), v.cuda(), starts, want_lse=True,
                              out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref, ref_lse = _oracle_segments(q, k, v, starts, hq, hkv)
    got = t2n(out)
    # K1 rounds P to bf16 before P.V: with a few keys carrying the weight the rounding does
    # not average out, so the max-norm bound is one bf16 unit (2^-8) and 2e-3 holds per head
    # in Frobenius norm — the bounds of test_fullsize_gpu (measured 2.2e-3 max-norm
    # on the rising case, the same floor as the random every-row check)
    for h in range(hq):
        for a, b in zip(starts[:-1], starts[1:]):
            assert normwise(got[a:b, h], ref[a:b, h]) <= 2.0 ** -8, ("K1", h, a)
            fro = np.linalg.norm(got[a:b, h] - ref[a:b, h]) / np.linalg.norm(ref[a:b, h])
            assert fro <= BF16_TOL, ("K1 Frobenius", h, a, fro)
    np.testing.assert_allclose(t2n(lse), ref_lse, atol=BF16_TOL, rtol=0)
    # ---- K2 (decode, l_q = 1) and K2q (query encode, l_q = 32, own tail) over a paged cache
    L, page = 5000, 128
    pps = -(-L // page)
    kc, vc = _rising(L, hkv, d, amp, gen, direction), torch.randn(L, hkv, d, generator=gen).bfloat16()
    kp = torch.zeros((pps, hkv, page, d), dtype=torch.bfloat16, device="cuda")
    vp = torch.zeros_like(kp)
    table = torch.arange(pps, dtype=torch.int32, device="cuda").view(1, pps)
    ops.kv_write(kc.cuda(), vc.cuda(), kp, vp, table[0].contiguous(), 0)
    kv_len = torch.tensor([L], dtype=torch.int32, device="cuda")
    for lq, own_tail in ((1, 0), (32, 32)):
        qd = _sharp_queries(lq, hq, d, gen).view(1, lq, hq, d)
        o, l = ops.phase2_partial(qd.cuda(), kp, vp, table, kv_len, L, own_tail=own_tail)
        torch.cuda.synchronize()
        for h in range(hq):
            kk = kc[:, h // G].float().numpy().astype(np.float64)
            vv = vc[:, h // G].float().numpy().astype(np.float64)
            keep = "full"
            if own_tail:
                keep = np.ones((lq, L), dtype=bool)
                keep[:, L - own_tail:] = O.causal_keep(lq, own_tail)
            ro, rl = O.partial_attention(qd[0, :, h].float().numpy().astype(np.float64), kk, vv, keep)
            assert normwise(t2n(o)[0, :, h], ro) <= BF16_TOL, ("K2", lq, h)
            np.testing.assert_allclose(t2n(l)[0, :, h], rl, atol=BF16_TOL, rtol=0)


def test_known_answers_on_the_kernels(ops):
    """SPEC's closed-form answers (tests/test_oracle.py checks them on the oracle) through the
    product kernels: the 2 x 2 analytic causal attention on K1 — identity q, k,
    v in the first two of 128 dimensions, so row 0 = v0 and row 1 = (v0 + e v1) / (1 + e) with
    e = exp(1 / sqrt(d)) — and the ln 2 lse shift of a duplicated key set on K2
    decode, K2q query encode and the fp32 check mode, output unchanged."""
    d = 128
    x = torch.zeros(2, 1, d)
    x[0, 0, 0] = x[1, 0, 1] = 1.0
    xb = x.bfloat16().cuda()
    out, lse = ops.phase1_fwd(xb, xb, xb, [0, 2], want_lse=True, out_dtype=torch.float32)
    torch.cuda.synchronize()
    e = float(np.exp(1 / np.sqrt(d)))
    ref = np.zeros((2, d))
    ref[0, 0] = 1.0
    ref[1, 0], ref[1, 1] = 1 / (1 + e), e / (1 + e)
    np.testing.assert_allclose(t2n(out)[:, 0], ref, atol=BF16_TOL)
    assert float(out[0, 0, 0]) == 1.0  # one visible key: P = 1 exactly
    np.testing.assert_allclose(t2n(lse)[0], [1 / np.sqrt(d), np.log(1 + e)], atol=BF16_TOL)
    # duplicated keys: the same cache twice -> lse + ln 2, same output
    gen = torch.Generator().manual_seed(2)
    n, hq, hkv, page = 1000, 8, 2, 64
    for dtype, lq, tol in ((torch.bfloat16, 1, BF16_TOL), (torch.bfloat16, 32, BF16_TOL),
                           (torch.float32, 1, 1e-5)):
        k = torch.randn(n, hkv, d, generator=gen).to(dtype)
        v = torch.randn(n, hkv, d, generator=gen).to(dtype)
        q = torch.randn(1, lq, hq, d, generator=gen).to(dtype).cuda()
        res = []
        for reps in (1, 2):
            rows = n * reps
            pps = -(-rows // page)
            kp = torch.zeros((pps, hkv, page, d), dtype=dtype, device="cuda")
            vp = torch.zeros_like(kp)
            table = torch.arange(pps, dtype=torch.int32, device="cuda").view(1, pps)
            ops.kv_write(k.repeat(reps, 1, 1).cuda(), v.repeat(reps, 1, 1).cuda(), kp, vp,
                         table[0].contiguous(), 0)
            kv_len = torch.tensor([rows], dtype=torch.int32, device="cuda")
            res.append(ops.phase2_partial(q, kp, vp, table, kv_len, rows))
        torch.cuda.synchronize()
        (o1, l1), (o2, l2) = res
        assert normwise(t2n(o2), t2n(o1)) <= tol, (dtype, lq)
        np.testing.assert_allclose(t2n(l2) - t2n(l1), np.log(2), atol=tol)


def test_phase2_workspace_reuse_across_shapes(ops):
    """One workspace, alternating shapes and split counts (query encode -> decode -> batch):
    the word-mode fix-up's epochs and words must never pick up a stale word of another
    layout (the library re-zeroes the workspace on a shape change)."""
    g = torch.Generator().manual_seed(9)
    hq, hkv, d, ps = 8, 2, 128, 64
    L = 3000
    pages = -(-L // ps)
    kp = torch.randn(2 * pages, hkv, ps, d, generator=g).to(torch.bfloat16).cuda()
    vp = torch.randn(2 * pages, hkv, ps, d, generator=g).to(torch.bfloat16).cuda()
    table = torch.arange(2 * pages, dtype=torch.int32).view(2, pages).cuda()
    ws = ops.Phase2Workspace()
    ref = {}
    for it in range(3):
        for B, lq, splits in ((1, 4, 12), (1, 1, 16), (2, 1, 9), (1, 1, 5), (2, 3, 0)):
            q = torch.randn(B, lq, hq, d, generator=torch.Generator().manual_seed(B * 10 + lq)).to(
                torch.bfloat16).cuda()
            kv_len = torch.full((B,), L, dtype=torch.int32).cuda()
            out, lse = ops.phase2_partial(q, kp, vp, table[:B], kv_len, L, n_splits=splits,
                                          workspace=ws)
            key = (B, lq, splits)
            if it == 0:
                # independent check: a fresh workspace per call
                o2, l2 = ops.phase2_partial(q, kp, vp, table[:B], kv_len, L, n_splits=splits,
                                            workspace=ops.Phase2Workspace())
                assert torch.equal(out, o2) and torch.equal(lse, l2), key
                ref[key] = (out.clone(), lse.clone())
            else:
                assert torch.equal(out, ref[key][0]) and torch.equal(lse, ref[key][1]), (it, key)


def test_merge_matches_reference(ops, golden_dir):
    g = np.load(f"{golden_dir}/attention.npz")
    outs = torch.from_numpy(g["merge_outs"]).cuda()
    lses = torch.from_numpy(g["merge_lses"].astype(np.float32)).cuda()
    out, lse = ops.merge(outs, lses)
    np.testing.assert_allclose(t2n(out), g["merge_out"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(t2n(lse), g["merge_lse"], rtol=1e-6)
    # a part with lse = -inf (an empty split) is skipped
    lses2 = torch.cat([lses, torch.full_like(lses[:1], -float("inf"))])
    outs2 = torch.cat([outs, torch.full_like(outs[:1], 123.0)])
    out2, lse2 = ops.merge(outs2, lses2)
    assert torch.allclose(out2, out) and torch.allclose(lse2, lse)
    # the packed wire format of the single all-gather ([rows*d out | rows lse] per part)
    # merges bit-identically to the separate tensors
    P, rows, d = outs.shape
    packed = torch.cat([outs.reshape(P, -1), lses.reshape(P, -1)], dim=1).contiguous()
    out3, lse3 = ops.merge_packed(packed, rows, d)
    assert torch.equal(out3, out) and torch.equal(lse3, lse)
    buf, po, pl = ops.packed_partial(rows, d, outs.device)
    assert po.data_ptr() == buf.data_ptr() and pl.data_ptr() == buf.data_ptr() + rows * d * 4


def test_phase1_anchor_dedup_bit_exact(ops):
    """with first-block anchors the deduplicated launch equals the full one."""
    hq, hkv, d, a = 8, 2, 128, 384
    own = [640, 512, 700]
    seg = [0]
    for i, o in enumerate(own):
        seg.append(seg[-1] + o + (a if i else 0))
    rows = seg[-1]
    q = torch.randn(rows, hq, d).to(torch.bfloat16)
    k = torch.randn(rows, hkv, d).to(torch.bfloat16)
    v = torch.randn(rows, hkv, d).to(torch.bfloat16)
    for s in range(1, len(own)):  # anchor rows = block 0's first a rows
        for t in (q, k, v):
            t[seg[s]:seg[s] + a] = t[:a]
    q, k, v = q.cuda(), k.cuda(), v.cuda()
    full, full_l = ops.phase1_fwd(q, k, v, seg, want_lse=True)
    dd, dd_l = ops.phase1_fwd(q, k, v, seg, want_lse=True, dedup_anchor_rows=a)
    torch.cuda.synchronize()
    assert torch.equal(full, dd) and torch.equal(full_l, dd_l)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_fused_prologue_equals_rope_plus_kv_write(ops, dtype):
    """rope_qkv == rope(q), rope(k) and kv_write of the cached rows, bit-exact."""
    rows, hq, hkv, d, page = 300, 8, 2, 128, 64
    rng = np.random.default_rng(11)
    q = torch.randn(rows, hq, d).to(dtype).cuda()
    k = torch.randn(rows, hkv, d).to(dtype).cuda()
    v = torch.randn(rows, hkv, d).to(dtype).cuda()
    pos = torch.from_numpy(rng.integers(0, 1 << 20, rows)).cuda()
    cache_rows = torch.full((rows,), -1, dtype=torch.int64)
    cache_rows[100:] = torch.arange(200)  # the last 200 rows are "own" rows
    cache_rows = cache_rows.cuda()
    n_pages = 5
    table = torch.tensor([3, 1, 4, 0], dtype=torch.int32).cuda()
    kp = torch.zeros((n_pages, hkv, page, d), dtype=dtype, device="cuda")
    vp = torch.zeros_like(kp)
    qo, ko = ops.rope_qkv(q, k, v, pos, cache_rows=cache_rows, k_pages=kp, v_pages=vp,
                          page_table=table)
    q_ref = ops.rope(q, pos)
    k_ref = ops.rope(k, pos)
    kp2, vp2 = torch.zeros_like(kp), torch.zeros_like(vp)
    ops.kv_write(k_ref[100:], v[100:], kp2, vp2, table, 0)
    torch.cuda.synchronize()
    assert torch.equal(qo, q_ref) and torch.equal(ko, k_ref)
    assert torch.equal(kp, kp2) and torch.equal(vp, vp2)


def test_fused_prologue_vector_and_scalar_forms_agree(ops):
    """The bf16 prologue runs 16-byte accesses when every row is 16-byte aligned, else the
    one-pair-per-thread kernel: a q whose storage starts one element off (the scalar form)
    gives the same bits as the aligned copy (the vector form), pages included."""
    rows, hq, hkv, d, page = 260, 8, 2, 128, 64
    rng = np.random.default_rng(12)
    base = torch.randn(rows * hq * d + 1).bfloat16().cuda()
    q_odd = base[1:].view(rows, hq, d)  # 2-byte aligned only
    q_al = q_odd.clone()
    k = torch.randn(rows, hkv, d).bfloat16().cuda()
    v = torch.randn(rows, hkv, d).bfloat16().cuda()
    pos = torch.from_numpy(rng.integers(0, 1 << 17, rows)).cuda()
    cache_rows = torch.full((rows,), -1, dtype=torch.int64)
    cache_rows[60:] = torch.arange(200)
    cache_rows = cache_rows.cuda()
    table = torch.tensor([2, 0, 3, 1], dtype=torch.int32).cuda()
    outs = []
    for q in (q_odd, q_al):
        kp = torch.zeros((4, hkv, page, d), dtype=torch.bfloat16, device="cuda")
        vp = torch.zeros_like(kp)
        qo, ko = ops.rope_qkv(q, k, v, pos, cache_rows=cache_rows, k_pages=kp, v_pages=vp,
                              page_table=table)
        outs.append((qo, ko, kp, vp))
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(*outs))
    assert torch.equal(outs[1][0], ops.rope(q_al, pos))


@pytest.mark.parametrize("d,hq,hkv,dtype", [(128, 8, 2, torch.bfloat16), (64, 4, 4, torch.bfloat16),
                                            (64, 4, 2, torch.float32)])
def test_phase1_query_range(ops, d, hq, hkv, dtype):
    """star_phase1_fwd_range == causal_attention(q[b:e], k[:e], v[:e], q_offset=b)
    (ss/attention.py:109-122): parts of a segment reassemble the whole-segment encode
    (bit-exact on the tensor-core path) and match the oracle's q_offset form."""
    m = 640
    q = ops.prng_fill((m, hq, d), 31, 1, 1.0, dtype, "cuda")
    k = ops.prng_fill((m, hkv, d), 32, 1, 1.0, dtype, "cuda")
    v = ops.prng_fill((m, hkv, d), 33, 1, 1.0, dtype, "cuda")
    full, full_lse = ops.phase1_fwd(q, k, v, [0, m], want_lse=True)
    got = torch.zeros_like(full)
    lse = torch.zeros((hq, m), dtype=torch.float32, device="cuda")
    for b, e in ((0, 256), (256, 384), (384, m)):
        ops.phase1_fwd_range(q, k, v, b, e, out=got, lse=lse)
    torch.cuda.synchronize()
    if dtype == torch.bfloat16:
        assert torch.equal(got, full) and torch.equal(lse, full_lse)
    G = hq // hkv
    qn, kn, vn = (t2n(t).astype(np.float64) for t in (q, k, v))
    for h in (0, hq - 1):
        ro, rl = O.causal_attention_lse(qn[256:384, h], kn[:384, h // G], vn[:384, h // G],
                                        q_offset=256)
        g = t2n(got[256:384, h])
        if dtype == torch.float32:
            np.testing.assert_allclose(g, ro, rtol=1e-5, atol=1e-6)
        else:
            assert normwise(g, ro) <= BF16_OUT_TOL
        np.testing.assert_allclose(t2n(lse[h, 256:384]), rl, atol=BF16_TOL)
    if dtype == torch.bfloat16:
        from paper_2411_17116_b200.errors import ConfigError
        with pytest.raises(ConfigError):
            ops.phase1_fwd_range(q, k, v, 100, 300, out=got)  # not a whole q tile


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_phase1_more_segments_than_one_launch(ops, dtype):
    """A context with more blocks than one launch's segment table (kMaxSegments = 64) runs
    as several launches: every segment equals its own single-segment encode (bit-exact),
    and anchor dedup across the launch boundary equals the full encode."""
    hq, hkv, d, a = 4, 2, 64, 128
    n = 70
    own = [128 + 64 * (i % 3) for i in range(n)]
    seg = [0]
    for i, o in enumerate(own):
        seg.append(seg[-1] + o + (a if i else 0))
    rows = seg[-1]
    q = ops.prng_fill((rows, hq, d), 41, 1, 1.0, dtype, "cuda")
    k = ops.prng_fill((rows, hkv, d), 42, 1, 1.0, dtype, "cuda")
    v = ops.prng_fill((rows, hkv, d), 43, 1, 1.0, dtype, "cuda")
    for s in range(1, n):  # first-block anchors
        for t in (q, k, v):
            t[seg[s]:seg[s] + a] = t[:a]
    full, full_l = ops.phase1_fwd(q, k, v, seg, want_lse=True)
    for s in (0, 1, 63, 64, 69):
        b, e = seg[s], seg[s + 1]
        one, one_l = ops.phase1_fwd(q[b:e].contiguous(), k[b:e].contiguous(), v[b:e].contiguous(),
                                    [0, e - b], want_lse=True)
        assert torch.equal(full[b:e], one), s
        assert torch.equal(full_l[:, b:e], one_l), s
    if dtype == torch.bfloat16:
        dd, dd_l = ops.phase1_fwd(q, k, v, seg, want_lse=True, dedup_anchor_rows=a)
        torch.cuda.synchronize()
        assert torch.equal(full, dd) and torch.equal(full_l, dd_l)


@pytest.mark.parametrize("dtype,B,rows", [(torch.bfloat16, 1, 1), (torch.float32, 1, 3),
                                          (torch.bfloat16, 4, 1), (torch.bfloat16, 3, 2)])
def test_kv_append_equals_rope_and_page_write(ops, dtype, B, rows):
    """star_kv_append (the graph-safe decode append): rotated q, and rotated k / raw v at the
    rows each sequence's DEVICE counter names, bit-exact against rope + kv_write at host rows;
    counters advanced by `rows`."""
    hq, hkv, d, page = 8, 2, 128, 64
    pps = 3
    n = B * rows
    q = torch.randn(n, hq, d).to(dtype).cuda()
    k = torch.randn(n, hkv, d).to(dtype).cuda()
    v = torch.randn(n, hkv, d).to(dtype).cuda()
    pos = torch.randint(1000, 1200, (n,), dtype=torch.int64).cuda()
    start = [37, 63, 0, 120][:B]  # crosses a page boundary for sequence 1
    kv_len = torch.tensor(start, dtype=torch.int32).cuda()
    table = torch.randperm(B * pps).to(torch.int32).view(B, pps).cuda()
    kp = torch.zeros((B * pps, hkv, page, d), dtype=dtype, device="cuda")
    vp = torch.zeros_like(kp)
    qo = ops.kv_append(q, k, v, pos, kv_len, kp, vp, table)
    # through a cos/sin table of (some of) the positions: bit-identical
    kv_len_t = torch.tensor(start, dtype=torch.int32).cuda()
    kp_t, vp_t = torch.zeros_like(kp), torch.zeros_like(vp)
    tab = ops.RopeTable(1000, 100, d, 10000.0, "cuda")  # positions >= 1100 form angles in place
    qo_t = ops.kv_append(q, k, v, pos, kv_len_t, kp_t, vp_t, table, table=tab)
    kp2, vp2 = torch.zeros_like(kp), torch.zeros_like(vp)
    q_ref = ops.rope(q, pos)
    k_ref = ops.rope(k, pos)
    for b in range(B):
        sl = slice(b * rows, (b + 1) * rows)
        ops.kv_write(k_ref[sl], v[sl], kp2, vp2, table[b].contiguous(), start[b])
    torch.cuda.synchronize()
    assert torch.equal(qo, q_ref) and torch.equal(qo_t, q_ref)
    assert torch.equal(kp, kp2) and torch.equal(vp, vp2)
    assert torch.equal(kp_t, kp2) and torch.equal(vp_t, vp2)
    assert kv_len.tolist() == [s + rows for s in start] == kv_len_t.tolist()


@pytest.mark.parametrize("B,hq,hkv,d,starts", [
    (1, 32, 8, 128, [16383]),          # Llama-8B heads, the new row ends a 64-key tile
    (1, 32, 8, 128, [16384]),          # the new row opens a new page / tile
    (3, 8, 2, 128, [37, 4095, 200]),   # batch, ragged lengths
    (2, 8, 8, 64, [129, 0]),           # MHA, head_dim 64, an empty cache (first row)
])
@pytest.mark.parametrize("use_table", ["table", "none", "cur"])
def test_phase2_decode_equals_append_then_k2(ops, B, hq, hkv, d, starts, use_table):
    """star_phase2_decode (RoPE + append inside K2, one launch) is BIT-IDENTICAL to
    star_kv_append followed by star_phase2_partial: same pages written, same (out, lse); the
    counters are untouched until star_decode_advance, which adds 1 to each and 1 to each
    position.  append=False (a rank that only rotates q) equals rope + K2."""
    page = 128
    maxk = max(starts) + 64
    pps = -(-maxk // page)
    torch.manual_seed(7)
    q = torch.randn(B, hq, d).bfloat16().cuda()
    k = torch.randn(B, hkv, d).bfloat16().cuda()
    v = torch.randn(B, hkv, d).bfloat16().cuda()
    pos = torch.tensor([s + 11 for s in starts], dtype=torch.int64).cuda()
    table = torch.randperm(B * pps).to(torch.int32).view(B, pps).cuda()
    kp = ops.prng_fill((B * pps, hkv, page, d), 3, 1, 1.0, torch.bfloat16, torch.device("cuda"))
    vp = ops.prng_fill((B * pps, hkv, page, d), 4, 1, 1.0, torch.bfloat16, torch.device("cuda"))
    tab = ops.RopeTable(min(starts) + 11, maxk, d, 10000.0, "cuda") if use_table == "table" else None
    rope = None
    if use_table == "cur":  # DecodeRope: cos/sin at the current positions, primed on the device
        rope = ops.DecodeRope(min(starts) + 11, maxk, d, 10000.0, B, "cuda")
        rope.prime(pos)
        tab = rope.table
    # reference: append kernel + K2
    kp_r, vp_r = kp.clone(), vp.clone()
    kl_r = torch.tensor(starts, dtype=torch.int32).cuda()
    qr = ops.kv_append(q.view(B, hq, d), k, v, pos, kl_r, kp_r, vp_r, table, table=tab)
    o_r, l_r = ops.phase2_partial(qr.view(B, 1, hq, d), kp_r, vp_r, table, kl_r, maxk)
    # fused
    kl = torch.tensor(starts, dtype=torch.int32).cuda()
    o, l = ops.phase2_decode(q, k, v, pos, kp, vp, table, kl, maxk, table=rope or tab)
    torch.cuda.synchronize()
    assert torch.equal(kp, kp_r) and torch.equal(vp, vp_r)
    assert torch.equal(o, o_r) and torch.equal(l, l_r)
    assert kl.tolist() == starts
    pos2 = pos.clone()
    ops.decode_advance(kl, pos2, rope=rope)
    torch.cuda.synchronize()
    assert kl.tolist() == [s + 1 for s in starts] and torch.equal(pos2, pos + 1)
    if rope is not None:  # cur now holds the table rows of the advanced positions
        for b in range(B):
            assert torch.equal(rope.cur[b], rope.table.cs[int(pos2[b]) - rope.table.pos0])
    # rotate-only (no append) == rope + K2 over the unchanged cache
    kl0 = torch.tensor(starts, dtype=torch.int32).cuda()
    if rope is not None:
        rope.prime(pos)
    o2, l2 = ops.phase2_decode(q, None, None, pos, kp, vp, table, kl0, maxk, table=rope or tab,
                               append=False)
    o3, l3 = ops.phase2_partial(ops.rope(q, pos).view(B, 1, hq, d), kp, vp, table, kl0, maxk)
    torch.cuda.synchronize()
    assert torch.equal(o2, o3) and torch.equal(l2, l3)


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("n_splits", [0, 1])
def test_decode_chain_reads_the_current_counter(ops, fused, n_splits):
    """K2 is launched as a programmatic dependent (PDL) of the kernel before it, and the one
    before it may have just written the row counter: star_kv_append triggers its dependents at
    entry and bumps kv_len at its end; star_decode_advance bumps every counter.  K2 must read
    kv_len after griddepcontrol.wait — through a const __restrict__ pointer the compiler had
    hoisted the load above it.  T chained steps on one stream with a primed workspace (so
    every K2 launch is PDL), each step's (out, lse) equal, bit for bit, to K2 rerun on that
    step's state after a device sync.  n_splits = 1 is a plain (not cooperative) launch, the
    one that overlaps its predecessor the most."""
    B, hq, hkv, d, page, T = 1, 32, 8, 128, 128, 24
    start = 3000
    maxk = start + T + 64
    pps = -(-maxk // page)
    dev = torch.device("cuda")
    torch.manual_seed(5)
    q = torch.randn(B, hq, d).bfloat16().cuda()
    k = torch.randn(B, hkv, d).bfloat16().cuda()
    v = torch.randn(B, hkv, d).bfloat16().cuda()
    table = torch.arange(pps, dtype=torch.int32, device=dev).view(B, pps)
    kp = ops.prng_fill((pps, hkv, page, d), 3, 1, 1.0, torch.bfloat16, dev)
    vp = ops.prng_fill((pps, hkv, page, d), 4, 1, 1.0, torch.bfloat16, dev)
    pos = torch.tensor([start + 11], dtype=torch.int64, device=dev)
    kl = torch.tensor([start], dtype=torch.int32, device=dev)
    rope = ops.DecodeRope(start + 11, T + 8, d, 10000.0, B, dev) if fused else None
    ws = ops.Phase2Workspace()
    ns = n_splits
    ops.phase2_partial(q.view(B, 1, hq, d), kp, vp, table, kl, maxk, n_splits=ns, workspace=ws)  # prime
    if fused:
        rope.prime(pos)
    steps = []
    for _ in range(T):
        if fused:
            o, l = ops.phase2_decode(q, k, v, pos, kp, vp, table, kl, maxk, table=rope,
                                     n_splits=ns, workspace=ws)
            ops.decode_advance(kl, pos, rope=rope)
            steps.append((None, o, l))
        else:
            qr = ops.kv_append(q, k, v, pos, kl, kp, vp, table)
            o, l = ops.phase2_partial(qr.view(B, 1, hq, d), kp, vp, table, kl, maxk, n_splits=ns,
                                      workspace=ws)
            pos.add_(1)
            steps.append((qr, o, l))
    torch.cuda.synchronize()
    assert int(kl[0]) == start + T
    for t, (qr, o, l) in enumerate(steps):
        kl_t = torch.tensor([start + t + 1], dtype=torch.int32, device=dev)
        if qr is None:  # the fused step attended over its own new row: rerun unfused on it
            qr = ops.rope(q, torch.tensor([start + 11 + t], dtype=torch.int64, device=dev))
        o2, l2 = ops.phase2_partial(qr.view(B, 1, hq, d), kp, vp, table, kl_t, maxk, n_splits=ns,
                                    workspace=ws)
        torch.cuda.synchronize()
        assert torch.equal(o, o2) and torch.equal(l, l2), t


def test_phase2_decode_exchange_equals_unfused(ops):
    """The fused decode step through the one-kernel peer exchange (2 ranks' boxes on one GPU,
    one stream per rank, grids small enough to be co-resident as on separate GPUs) equals the
    fused decode partials merged by K3, bit for bit; rank 1 (the query rank) appends."""
    from paper_2411_17116_b200.dist import local_peer_exchanges

    B, hq, hkv, d, page, splits = 1, 32, 8, 128, 128, 4
    rows = [5000, 7000]
    maxk = max(rows) + 64
    pps = -(-maxk // page)
    dev = torch.device("cuda")
    torch.manual_seed(3)
    q = torch.randn(B, hq, d).bfloat16().cuda()
    k = torch.randn(B, hkv, d).bfloat16().cuda()
    v = torch.randn(B, hkv, d).bfloat16().cuda()
    pos = torch.tensor([rows[1] + 3], dtype=torch.int64).cuda()
    tab = ops.RopeTable(int(pos[0]), 8, d, 10000.0, "cuda")
    pools = [(ops.prng_fill((pps, hkv, page, d), 10 + r, 1, 1.0, torch.bfloat16, dev),
              ops.prng_fill((pps, hkv, page, d), 20 + r, 1, 1.0, torch.bfloat16, dev),
              torch.arange(pps, dtype=torch.int32, device=dev).view(1, -1)) for r in range(2)]
    refs = []
    for r in range(2):
        kp, vp, tb = pools[r]
        kl = torch.tensor([rows[r]], dtype=torch.int32, device=dev)
        refs.append(ops.phase2_decode(q, k, v, pos, kp.clone(), vp.clone(), tb, kl, maxk,
                                      table=tab, append=r == 1, n_splits=splits))
    exs = local_peer_exchanges(2, hq, hkv, d, dev)
    streams = [torch.cuda.Stream() for _ in range(2)]
    kls = [torch.tensor([rows[r]], dtype=torch.int32, device=dev) for r in range(2)]
    torch.cuda.synchronize()
    outs = [None, None]
    for r in range(2):
        kp, vp, tb = pools[r]
        with torch.cuda.stream(streams[r]):
            outs[r] = exs[r].decode_exchange(q, k, v, pos, kp, vp, tb, kls[r], maxk, 10000.0, tab,
                                             append=r == 1, n_splits=splits,
                                             workspace=ops.Phase2Workspace())
    torch.cuda.synchronize()
    o_ref, l_ref = ops.merge(torch.stack([refs[0][0].view(-1, d), refs[1][0].view(-1, d)]),
                             torch.stack([refs[0][1].view(-1), refs[1][1].view(-1)]))
    torch.cuda.synchronize()
    for o, l in outs:
        assert torch.equal(o.view(-1, d), o_ref.view(-1, d))
        assert torch.equal(l.view(-1), l_ref.view(-1))
