"""Fused phase-2 exchange (PeerExchange: K2 epilogue -> every rank's box -> K3x) on the B200.

Several ranks' boxes live in ONE process here (dist.local_peer_exchanges): the kernels,
box layout, epochs and flags are the production ones; only the IPC mapping is skipped
(tests/test_dist_gpu.py covers that with two processes).  Checks:
  * bit-exact against the unfused path (K2 into local buffers, then K3 over the stacked
    partials) — the pushed values are the same floats, the merge is the same arithmetic;
  * the merged result against the CPU oracle's partial_attention + merge_partials over
    the union of the ranks' keys (ss/attention.py:125-173, ss/sim.py:178-213);
  * empty ranks (lse = -inf, skipped like ss/sim.py:193-194), alternating epochs and
    changing shapes (query encode then decode steps) in one box.
"""

import numpy as np
import pytest
import torch

from oracle import star_oracle as O

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-3


@pytest.fixture(scope="module")
def mods():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2411_17116_b200 import dist as D
    from paper_2411_17116_b200 import ops
    return ops, D


def _rank_caches(lens, hkv, d, dtype, page_size, seed):
    """One paged cache per rank (None for an empty rank)."""
    g = torch.Generator().manual_seed(seed)
    caches = []
    for L in lens:
        if L == 0:
            caches.append(None)
            continue
        k = torch.randn(L, hkv, d, generator=g).to(dtype)
        v = torch.randn(L, hkv, d, generator=g).to(dtype)
        pages = (L + page_size - 1) // page_size
        kp = torch.zeros((pages + 2, hkv, page_size, d), dtype=dtype, device="cuda")
        vp = torch.zeros_like(kp)
        table = torch.randperm(pages + 2, generator=g)[:pages].to(torch.int32).cuda()
        caches.append((k, v, kp, vp, table))
    return caches


def _write(ops, caches):
    for c in caches:
        if c is not None:
            k, v, kp, vp, table = c
            ops.kv_write(k.cuda(), v.cuda(), kp, vp, table, 0)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("world,lens,hq,hkv,d,splits,lq_query", [
    # l_q = 32 at Llama-8B heads: the query encode runs on the tcgen05 K2q kernel
    (3, [4096, 1000, 2500], 32, 8, 128, 0, 32),
    (3, [4096, 1000, 2500], 32, 8, 128, 0, 4),    # Llama-8B heads, auto splits (fix-up pushes)
    (4, [700, 0, 3000, 64], 8, 2, 64, 1, 4),      # one split per group (epilogue pushes), empty rank
    (2, [20000, 9000], 8, 8, 128, 0, 4),
    (8, [16384, 9000, 16384, 0, 5000, 16384, 700, 16384], 32, 8, 128, 0, 4),  # a full node
])
def test_exchange_matches_unfused_and_oracle(mods, dtype, world, lens, hq, hkv, d, splits,
                                             lq_query):
    ops, D = mods
    page_size = 64
    caches = _rank_caches(lens, hkv, d, dtype, page_size, seed=world * 7 + hq)
    _write(ops, caches)
    exs = D.local_peer_exchanges(world, lq_query * hq, hkv, d, "cuda")
    g = torch.Generator().manual_seed(5)
    # a query encode (own tail on the last rank), then two 1-row decode steps
    for step, (lq, tail) in enumerate([(lq_query, lq_query), (1, 0), (1, 0)]):
        q = torch.randn(1, lq, hq, d, generator=g).to(dtype)
        qd = q.cuda()
        ref_o, ref_l = [], []
        for r, c in enumerate(caches):
            own = tail if r == world - 1 else 0
            if c is None:
                o = torch.zeros(lq * hq, d, device="cuda")
                s = torch.full((lq * hq,), float("-inf"), device="cuda")
                exs[r].push(o, s, 1, lq, hq, hkv)
            else:
                k, v, kp, vp, table = c
                kv_len = torch.tensor([k.shape[0]], dtype=torch.int32, device="cuda")
                exs[r].push_partial(qd, kp, vp, table.view(1, -1), kv_len, k.shape[0],
                                    own_tail=own, n_splits=splits)
                o, s = ops.phase2_partial(qd, kp, vp, table.view(1, -1), kv_len, k.shape[0],
                                          own_tail=own, n_splits=splits)
                o, s = o.view(lq * hq, d), s.view(lq * hq)
            ref_o.append(o)
            ref_l.append(s)
        unfused, unfused_lse = ops.merge(torch.stack(ref_o), torch.stack(ref_l))
        for r in range(world):
            out, lse = exs[r].merge(1, lq, hq, hkv)
            assert torch.equal(out, unfused), (step, r)
            assert torch.equal(lse, unfused_lse), (step, r)
        # oracle: partial per non-empty rank, merged in ascending rank order
        G = hq // hkv
        got = out.view(lq, hq, d).cpu().numpy()
        got_lse = lse.view(lq, hq).cpu().numpy()
        for h in range(hq):
            parts = []
            qq = q[0, :, h].float().numpy().astype(np.float64)
            for r, c in enumerate(caches):
                if c is None:
                    continue
                k, v = c[0], c[1]
                kk = k[:, h // G].float().numpy().astype(np.float64)
                vv = v[:, h // G].float().numpy().astype(np.float64)
                own = tail if r == world - 1 else 0
                keep = "full"
                if own:
                    keep = np.ones((lq, kk.shape[0]), dtype=bool)
                    keep[:, kk.shape[0] - own:] = O.causal_keep(lq, own)
                parts.append(O.partial_attention(qq, kk, vv, keep))
            ro, rl = O.merge_partials([p[0] for p in parts], [p[1] for p in parts])
            if dtype == torch.float32:
                np.testing.assert_allclose(got[:, h], ro, rtol=1e-5, atol=1e-6)
                np.testing.assert_allclose(got_lse[:, h], rl, rtol=1e-6, atol=1e-5)
            else:
                err = np.abs(got[:, h] - ro).max() / np.abs(ro).max()
                assert err <= BF16_TOL, (step, h, err)
                np.testing.assert_allclose(got_lse[:, h], rl, atol=BF16_TOL)


def test_exchange_batched_decode(mods):
    """B = 4 sequences per rank (cfg5-style batch), 2 ranks, bf16 output of the merge."""
    ops, D = mods
    world, B, hq, hkv, d, page_size = 2, 4, 32, 8, 128, 64
    g = torch.Generator().manual_seed(11)
    lens = [[3000, 64, 5000, 700], [128, 4000, 1, 2200]]
    exs = D.local_peer_exchanges(world, B * hq, B * hkv, d, "cuda")
    q = torch.randn(B, 1, hq, d, generator=g).to(torch.bfloat16).cuda()
    parts = []
    for r in range(world):
        pps = (max(lens[r]) + page_size - 1) // page_size
        kp = torch.randn(B * pps, hkv, page_size, d, generator=g).to(torch.bfloat16).cuda()
        vp = torch.randn(B * pps, hkv, page_size, d, generator=g).to(torch.bfloat16).cuda()
        table = torch.randperm(B * pps, generator=g).to(torch.int32).view(B, pps).cuda()
        kv_len = torch.tensor(lens[r], dtype=torch.int32).cuda()
        exs[r].push_partial(q, kp, vp, table, kv_len, max(lens[r]))
        o, s = ops.phase2_partial(q, kp, vp, table, kv_len, max(lens[r]))
        parts.append((o.view(B * hq, d), s.view(B * hq)))
    ref, ref_lse = ops.merge(torch.stack([p[0] for p in parts]), torch.stack([p[1] for p in parts]),
                             out_dtype=torch.bfloat16)
    for r in range(world):
        out, lse = exs[r].merge(B, 1, hq, hkv, out_dtype=torch.bfloat16)
        assert torch.equal(out, ref) and torch.equal(lse, ref_lse)


def test_exchange_rejects_oversized_call(mods):
    ops, D = mods
    from paper_2411_17116_b200.errors import ShapeError

    exs = D.local_peer_exchanges(2, 8, 2, 64, "cuda")
    o = torch.zeros(16, 64, device="cuda")
    s = torch.zeros(16, device="cuda")
    with pytest.raises(ShapeError, match="box holds"):
        exs[0].push(o, s, 1, 4, 4, 2)


@pytest.mark.parametrize("world,splits,hq,hkv,lq_q,d", [(1, 0, 8, 2, 4, 128), (3, 2, 8, 2, 4, 128),
                                                        (2, 3, 8, 2, 4, 128), (8, 2, 8, 2, 4, 128),
                                                        (2, 2, 32, 8, 32, 128), (1, 0, 32, 8, 32, 128),
                                                        # MHA, d = 64, one query row: 64 output
                                                        # elements over 9 / 17 splits leave the
                                                        # last splits' fold slices empty
                                                        (2, 9, 2, 2, 1, 64), (3, 17, 2, 2, 1, 64)])
def test_fused_exchange_one_kernel(mods, world, splits, hq, hkv, lq_q, d):
    """star_phase2_exchange: partial + push + cross-rank merge in ONE K2 launch per rank
    (co-resident word-mode grid).  Ranks run on separate streams of one GPU with small grids
    (world x splits x hkv CTAs all resident), as they would on separate GPUs; bit-exact
    against the unfused K2 + K3 merge, and against plain K2 for one rank.  Ten steps, so a
    CTA with an empty fold slice arriving last (it must still carry the box epoch) shows up."""
    ops, D = mods
    ps = 64
    lens = [2000, 1500, 2600, 900, 3100, 1700, 2222, 1300][:world]
    caches = _rank_caches(lens, hkv, d, torch.bfloat16, ps, seed=21 + world)
    _write(ops, caches)
    exs = D.local_peer_exchanges(world, lq_q * hq, hkv, d, "cuda")
    streams = [torch.cuda.Stream() for _ in range(world)]
    g = torch.Generator().manual_seed(3)
    steps = [(lq_q, lq_q)] + [(1, 0)] * (2 if d == 128 else 9)
    for lq, tail in steps:
        q = torch.randn(1, lq, hq, d, generator=g).to(torch.bfloat16).cuda()
        torch.cuda.synchronize()
        outs = [None] * world
        for r, (k, v, kp, vp, table) in enumerate(caches):
            kv_len = torch.tensor([k.shape[0]], dtype=torch.int32, device="cuda")
            with torch.cuda.stream(streams[r]):
                outs[r] = exs[r].exchange(q, kp, vp, table.view(1, -1), kv_len, k.shape[0],
                                          own_tail=tail if r == world - 1 else 0,
                                          n_splits=splits, workspace=ops.Phase2Workspace())
        torch.cuda.synchronize()
        parts = []
        for r, (k, v, kp, vp, table) in enumerate(caches):
            kv_len = torch.tensor([k.shape[0]], dtype=torch.int32, device="cuda")
            o, s = ops.phase2_partial(q, kp, vp, table.view(1, -1), kv_len, k.shape[0],
                                      own_tail=tail if r == world - 1 else 0, n_splits=splits)
            parts.append((o.view(lq * hq, d), s.view(lq * hq)))
        if world == 1:
            ref, ref_lse = parts[0]
        else:
            ref, ref_lse = ops.merge(torch.stack([p[0] for p in parts]),
                                     torch.stack([p[1] for p in parts]))
        for r in range(world):
            o, s = outs[r]
            assert torch.equal(o.view(lq * hq, d), ref), (lq, r)
            assert torch.equal(s.view(lq * hq), ref_lse), (lq, r)


def test_epoch_counters_wrap(mods):
    """Box and word-mode epochs across the 32-bit wrap (0xFFFFFFFE -> 0xFFFFFFFF -> 2 -> 3):
    0 is skipped (it is the value of a zeroed word) and the parity keeps alternating."""
    ops, D = mods
    hq, hkv, d, ps = 8, 2, 128, 64
    caches = _rank_caches([3000, 2000], hkv, d, torch.bfloat16, ps, seed=77)
    _write(ops, caches)
    # two ranks in one process: the two-kernel path (K2 push + K3x); one rank: the one-kernel path
    for world in (2, 1):
        exs = D.local_peer_exchanges(world, hq, hkv, d, "cuda")
        for ex in exs:
            ex.own_box.view(torch.int32)[0] = -2  # 0xFFFFFFFE completed exchanges
        ws = [ops.Phase2Workspace() for _ in range(world)]
        g = torch.Generator().manual_seed(1)
        for step in range(4):
            q = torch.randn(1, 1, hq, d, generator=g).to(torch.bfloat16).cuda()
            parts = []
            for r in range(world):
                k, v, kp, vp, table = caches[r]
                kv_len = torch.tensor([k.shape[0]], dtype=torch.int32, device="cuda")
                if step == 0:  # push the word-mode group epochs to the wrap too
                    ops.phase2_partial(q, kp, vp, table.view(1, -1), kv_len, k.shape[0],
                                       workspace=ws[r])
                    torch.cuda.synchronize()
                    hdr = ws[r].buf.view(torch.int32)
                    hdr[2048:2048 + hkv] = -2
                o, s = ops.phase2_partial(q, kp, vp, table.view(1, -1), kv_len, k.shape[0],
                                          workspace=ops.Phase2Workspace())
                parts.append((o.view(hq, d), s.view(hq)))
                if world == 2:
                    exs[r].push_partial(q, kp, vp, table.view(1, -1), kv_len, k.shape[0],
                                        workspace=ws[r])
            if world == 2:
                ref, ref_lse = ops.merge(torch.stack([p[0] for p in parts]),
                                         torch.stack([p[1] for p in parts]))
                for r in range(world):
                    out, lse = exs[r].merge(1, 1, hq, hkv)
                    assert torch.equal(out, ref) and torch.equal(lse, ref_lse), (world, step, r)
            else:
                k, v, kp, vp, table = caches[0]
                kv_len = torch.tensor([k.shape[0]], dtype=torch.int32, device="cuda")
                out, lse = exs[0].exchange(q, kp, vp, table.view(1, -1), kv_len, k.shape[0],
                                           workspace=ws[0])
                assert torch.equal(out.view(hq, d), parts[0][0]), (world, step)
                assert torch.equal(lse.view(hq), parts[0][1]), (world, step)
        torch.cuda.synchronize()
        hdr0 = int(exs[0].own_box.view(torch.int32)[0].item()) & 0xFFFFFFFF
        assert hdr0 == 4, hdr0  # 0xFFFFFFFF, 2, 3, 4


def _random_exchange_cases(n):
    rng = np.random.default_rng(4242)
    cases = []
    for _ in range(n):
        world = int(rng.integers(1, 9))
        hq, hkv = [(32, 8), (8, 2), (8, 8), (16, 4)][rng.integers(4)]
        d = int(rng.choice([64, 128]))
        lq = int(rng.choice([1, 4, 8, 32]))
        lens = [0 if rng.random() < 0.2 else int(rng.integers(max(lq, 1), 9000)) for _ in range(world)]
        if not any(lens):
            lens[-1] = int(rng.integers(lq, 9000))
        splits = int(rng.choice([0, 0, 1, 2, 4]))
        dtype = torch.float32 if rng.random() < 0.3 else torch.bfloat16
        cases.append((dtype, world, lens, hq, hkv, d, splits, lq))
    return cases


@pytest.mark.parametrize("case", _random_exchange_cases(10))
def test_exchange_random_shapes(mods, case):
    """A seeded random sweep of the fused exchange (1-8 ranks, empty ranks, GQA 1-4, d 64/128,
    query encodes of 1-32 rows incl. the K2q path, explicit and automatic splits, fp32 and
    bf16): the same bit-exact and oracle checks as the fixed cases above."""
    dtype, world, lens, hq, hkv, d, splits, lq = case
    test_exchange_matches_unfused_and_oracle(mods, dtype, world, lens, hq, hkv, d, splits, lq)
