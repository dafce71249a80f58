"""Layout contract of the drop-in, bit-exact against the reference's golden vectors.

Covers partition / AnchorSpec / augment / star_model (ss/blocking.py:49-236,
ss/baselines.py:124-160) and the reference's config errors.  CPU only.
"""

import json
import os

import numpy as np
import pytest

import paper_2411_17116_b200 as S
from paper_2411_17116_b200.errors import ConfigError, ShapeError


@pytest.fixture(scope="module")
def blocking(golden_dir):
    with open(os.path.join(golden_dir, "blocking.json")) as f:
        return json.load(f)


def test_partition_matches_reference(blocking):
    for c in blocking["partition"]:
        p = S.partition(c["L"], c["b"], c["H"], allow_idle=c["allow_idle"])
        assert (p.num_blocks, p.num_hosts) == (c["num_blocks"], c["num_hosts"])
        assert list(p.host_assignment) == c["assignment"]
        assert [list(p.block_span(i)) for i in range(p.num_blocks)] == c["spans"]
        for h in range(p.num_hosts):
            assert p.blocks_of(h) == [i for i, o in enumerate(c["assignment"]) if o == h]


def test_augment_every_anchor_mode_matches_reference(blocking):
    assert len(blocking["augment"]) == len(S.CONTENT_MODES) * len(S.POSITION_MODES) * 3
    for c in blocking["augment"]:
        spec = S.AnchorSpec(c["content_mode"], c["position_mode"], c["anchor_len"],
                            c["constant_token_id"], c["token_range"])
        got = S.augment(S.partition(c["L"], c["b"], c["H"]), c["tokens"], spec, S.Prng(c["prng_seed"]))
        assert len(got) == len(c["blocks"])
        for bl, ref in zip(got, c["blocks"]):
            assert list(bl.token_ids) == ref["token_ids"]
            assert list(bl.position_ids) == ref["position_ids"]
            assert bl.anchor_prefix_len == ref["anchor_prefix_len"]
            assert bl.block_index == ref["block_index"]
            assert bl.own_positions == tuple(ref["position_ids"][ref["anchor_prefix_len"]:])


def test_star_model_matches_reference(blocking):
    for c in blocking["star_model"]:
        L, b, a, d, heads, lq, ng, H = c["args"]
        r = S.star_model(L, b, a, d, heads, lq, ng, H)
        assert r.to_json() == {k: c[k] for k in r.to_json()}


def test_spec_examples():
    # SPEC.md:221-223
    p = S.partition(10, 4)
    assert [p.block_span(i) for i in range(3)] == [(0, 4), (4, 8), (8, 10)]
    assert S.partition(8, 8).num_blocks == 1
    assert S.partition(128 * 1024, 32 * 1024).num_blocks == 4
    # SPEC.md:231-232
    toks = list(range(100, 108))
    bl = S.augment(S.partition(8, 4), toks, S.AnchorSpec(anchor_len=4))
    assert bl[1].position_ids == (0, 1, 2, 3, 4, 5, 6, 7)
    assert bl[1].token_ids == tuple(toks[:4] + toks[4:])
    bl = S.augment(S.partition(12, 4), list(range(12)), S.AnchorSpec(position_mode="previous_block"))
    assert bl[2].position_ids[:4] == (4, 5, 6, 7)
    # SPEC.md:399
    assert S.star_model(16, 4).phase1_pairs == 118 and S.global_pairs(16) == 136


def test_config_errors():
    with pytest.raises(ConfigError):
        S.partition(0, 4)
    with pytest.raises(ConfigError):
        S.partition(8, 0)
    with pytest.raises(ConfigError):
        S.partition(8, 4, 3)
    assert S.partition(8, 4, 3, allow_idle=True).host_assignment == (0, 1)
    with pytest.raises(ConfigError):
        S.AnchorSpec(content_mode="bogus")
    with pytest.raises(ConfigError):
        S.AnchorSpec(anchor_len=0)
    with pytest.raises(ConfigError):
        S.augment(S.partition(8, 4), list(range(8)), S.AnchorSpec(anchor_len=5))
    with pytest.raises(ConfigError):
        S.augment(S.partition(8, 4), list(range(7)), S.AnchorSpec())
    with pytest.raises(ShapeError):
        S.AugmentedBlock((1, 2), (0,), 0, 0)
    with pytest.raises(ConfigError):
        S.AnchorSpec.from_config({"anchor_len": 3, "extra": 1})
    assert S.AnchorSpec.from_config(S.AnchorSpec(anchor_len=3).to_config()) == S.AnchorSpec(anchor_len=3)


def test_sparsity_pattern_figure2():
    pat = S.sparsity_pattern(S.partition(5, 1), S.AnchorSpec())
    exp = np.zeros((6, 6), dtype=bool)
    for i in range(5):
        exp[i, i] = True
        exp[i, 0] = True
    exp[5, :] = True
    assert (pat == exp).all()


def test_ledger_csv_format():
    led = S.CommLedger()
    led.append(2, 0, 3, "partial_out", 64)
    led.append(2, 0, 3, "partial_lse", 1)
    assert led.to_csv() == "phase,src,dst,kind,scalar_count\n2,0,3,partial_out,64\n2,0,3,partial_lse,1\n"
    assert led.total(kinds=("partial_lse",)) == 1 and led.total(phase=1) == 0


def test_host_prng_matches_reference(golden_dir):
    g = np.load(os.path.join(golden_dir, "prng.npz"))
    for i, seed in enumerate(g["seeds"]):
        p = S.Prng(int(seed))
        assert [p.next_u64() for _ in range(64)] == [int(x) for x in g["u64"][i]]
    p = S.Prng(11)
    assert [p.randint_below(256) for _ in range(200)] == list(g["randint256"])
    assert S.Prng(12).sample_sorted(100, 10) == list(g["sample_sorted_100_10"])
    assert S.Prng(13).shuffle(range(20)) == list(g["shuffle_20"])


def _augmented_positions(L, b, a, G, rank):
    """Context row of every augmented row of `rank`'s blocks (first-block anchors)."""
    n = -(-L // b)
    pos, seg, own = [], [0], []
    for i in range(n):
        if min(i * G // n, G - 1) != rank:
            continue
        o = min(b, L - i * b)
        rows = list(range(a)) + list(range(i * b, i * b + o)) if i else list(range(o))
        pos += rows
        seg.append(seg[-1] + len(rows))
        own.append(o)
    return np.array(pos), seg, own


@pytest.mark.parametrize("G,rank", [(1, 0), (4, 0), (4, 2), (2, 1)])
def test_context_layout_copy_plan(G, rank):
    """pipeline.LayerEncodePlan.set_context_layout: every augmented row is filled exactly
    once, from the context row the reference's augment() puts there (ss/blocking.py:206-236);
    each distinct context row crosses host->device once, repeats are device copies."""
    from paper_2411_17116_b200 import pipeline

    L, b, a = 40, 8, 8
    pos, seg, own = _augmented_positions(L, b, a, G, rank)
    plan = pipeline.LayerEncodePlan.__new__(pipeline.LayerEncodePlan)
    plan.seg, plan.own = seg, own
    n_ctx = plan.set_context_layout(pos)
    uniq = np.unique(pos)
    assert n_ctx == len(uniq)
    filled = np.full(len(pos), -1)
    h2d_rows = 0
    for h, dd in zip(plan.h2d, plan.d2d):
        for r0, c0, m in h:
            filled[r0:r0 + m] = uniq[c0:c0 + m]
            h2d_rows += m
        for r0, src, m in dd:
            assert (filled[src:src + m] >= 0).all()  # the source rows already landed
            filled[r0:r0 + m] = filled[src:src + m]
    assert (filled == pos).all()
    assert h2d_rows == n_ctx


def test_pipeline_cut_points():
    """Host logic of the e2e pipeline's causal parts (pipeline._cuts): whole 128-row q tiles,
    sorted, covering [0, m); only the first and last segments are split."""
    from paper_2411_17116_b200 import pipeline

    for m in (16384, 32768, 1000, 130):
        for first in (False, True):
            for last in (False, True):
                cuts = pipeline._cuts(m, first, last)
                assert cuts[0] == 0 and cuts[-1] == m
                assert cuts == sorted(set(cuts))
                assert all(c % 128 == 0 for c in cuts[:-1])
                if not first and not last:
                    assert cuts == [0, m]
    assert pipeline._cuts(16384, True, False) == [0, 8192, 16384]
    assert pipeline._cuts(32768, False, True) == [0, 16384, 24576, 32768]
