"""Pin the CPU oracle to golden vectors produced by the unmodified reference.

Integer / layout items are compared bit-exactly; floating point at the
reference's own tolerances (1e-5 relative for 32-bit scalars).
"""

import json
import os

import numpy as np
import pytest

from oracle import star_oracle as O


def _load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name), allow_pickle=False)


def test_prng_streams(golden_dir):
    g = _load(golden_dir, "prng.npz")
    for i, seed in enumerate(g["seeds"]):
        p = O.OraclePrng(int(seed))
        assert [p.u64() for _ in range(64)] == [int(x) for x in g["u64"][i]]
        p = O.OraclePrng(int(seed))
        np.testing.assert_array_equal([p.unit() for _ in range(16)], g["floats"][i])
        np.testing.assert_array_equal(O.uniform_fill(O.OraclePrng(int(seed)), 7, 5, 0.25, np.float32),
                                      g["fill32"][i])
        np.testing.assert_array_equal(O.uniform_fill(O.OraclePrng(int(seed)), 7, 5, 0.25, np.float64),
                                      g["fill64"][i])
        # the random-access form equals the sequential one
        np.testing.assert_array_equal(O.counter_fill(int(seed), 35, 0.25).reshape(7, 5), g["fill64"][i])
    p = O.OraclePrng(3)
    p.u64(), p.u64()
    np.testing.assert_array_equal(O.uniform_fill(p, 3, 4, 1.0), g["fill_after2"])
    p = O.OraclePrng(11)
    assert [p.below(256) for _ in range(200)] == list(g["randint256"])
    assert O.OraclePrng(12).floyd_sorted(100, 10) == list(g["sample_sorted_100_10"])
    assert O.OraclePrng(13).permuted(range(20)) == list(g["shuffle_20"])


def test_rope(golden_dir):
    g = _load(golden_dir, "rope.npz")
    for n in "abc":
        y = O.rope(g[f"{n}_x"], g[f"{n}_pos"], float(g[f"{n}_theta"]))
        assert y.dtype == g[f"{n}_y"].dtype
        np.testing.assert_array_equal(y, g[f"{n}_y"])


@pytest.mark.parametrize("case", ["c0", "c1", "c2", "c3"])
def test_attention_cases(golden_dir, case):
    g = _load(golden_dir, "attention.npz")
    q, k, v, off = g[f"{case}_q"], g[f"{case}_k"], g[f"{case}_v"], int(g[f"{case}_off"])
    np.testing.assert_allclose(O.causal_attention(q, k, v, off), g[f"{case}_out"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(O.streaming_causal_attention(q, k, v, 3, off), g[f"{case}_stream3"],
                               rtol=1e-5, atol=1e-6)
    o, l = O.partial_attention(q, k, v, "causal", off)
    np.testing.assert_allclose(o, g[f"{case}_pc_out"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(l, g[f"{case}_pc_lse"], rtol=1e-6, atol=1e-6)
    o, l = O.partial_attention(q, k, v, "full")
    np.testing.assert_allclose(o, g[f"{case}_pf_out"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(l, g[f"{case}_pf_lse"], rtol=1e-6, atol=1e-6)


def test_tail_mask_and_merge(golden_dir):
    g = _load(golden_dir, "attention.npz")
    o, l = O.partial_attention(g["tail_q"], g["tail_k"], g["tail_v"], g["tail_keep"])
    np.testing.assert_allclose(o, g["tail_out"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(l, g["tail_lse"], rtol=1e-6, atol=1e-6)
    mo, ml = O.merge_partials(list(g["merge_outs"]), list(g["merge_lses"]))
    np.testing.assert_allclose(mo, g["merge_out"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(ml, g["merge_lse"], rtol=1e-12)
    # and equals one partial over the concatenation
    fo, fl = O.partial_attention(g["merge_q"], g["merge_k"], g["merge_v"], "full")
    np.testing.assert_allclose(mo, fo, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(ml, fl, rtol=1e-6)


def test_spec_known_answers():
    # SPEC.md:134 analytic 2x2 causal
    eye = np.eye(2, dtype=np.float64)
    out = O.causal_attention(eye, eye, eye)
    e = np.exp(1 / np.sqrt(2))
    np.testing.assert_allclose(out, [[1, 0], [1 / (1 + e), e / (1 + e)]], rtol=1e-12)
    # SPEC.md:143 duplicating the key set adds ln 2 to lse
    rng = np.random.default_rng(0)
    q, k, v = (rng.standard_normal((3, 8)) for _ in range(3))
    o1, l1 = O.partial_attention(q, k, v)
    o2, l2 = O.partial_attention(q, np.concatenate([k, k]), np.concatenate([v, v]))
    np.testing.assert_allclose(l2 - l1, np.log(2), rtol=1e-12)
    np.testing.assert_allclose(o1, o2, rtol=1e-12)
    # SPEC.md:399 analytic pair count
    assert O.star_pairs(16, 4) == 118 and 16 * 17 // 2 == 136


def test_blocking(golden_dir):
    with open(os.path.join(golden_dir, "blocking.json")) as f:
        g = json.load(f)
    for c in g["partition"]:
        p = O.plan_blocks(c["L"], c["b"], c["H"], c["allow_idle"])
        assert p.n == c["num_blocks"] and p.H == c["num_hosts"]
        assert list(p.owner) == c["assignment"]
        assert [list(p.span(i)) for i in range(p.n)] == c["spans"]
    for c in g["augment"]:
        spec = O.Anchor(c["content_mode"], c["position_mode"], c["anchor_len"],
                        c["constant_token_id"], c["token_range"])
        got = O.augmented_blocks(O.plan_blocks(c["L"], c["b"], c["H"]), c["tokens"], spec,
                                 O.OraclePrng(c["prng_seed"]))
        assert len(got) == len(c["blocks"])
        for (t, p_, a), ref in zip(got, c["blocks"]):
            assert list(t) == ref["token_ids"]
            assert list(p_) == ref["position_ids"]
            assert a == ref["anchor_prefix_len"]
    for c in g["star_model"]:
        L, b, a, d, heads, lq, ng, H = c["args"]
        assert O.star_pairs(L, b, a) == c["phase1_pairs"]
        assert O.star_comm(L, b, d, heads, lq, ng, H) == c["phase2_comm"]


SMALL = ["small_n2", "small_n5h2", "small_n4h4"]
TINY = ["tiny_s0", "tiny_s4", "tiny_s7"]
# every non-default anchor mode through the whole protocol (make_golden.py MODEL_CASES)
ANCHOR = ["anc_prev", "anc_randpos", "anc_prevpos", "anc_shuffled", "anc_randtok", "anc_const",
          "anc_none"]


def _run_case(golden_dir, name):
    g = _load(golden_dir, f"model_{name}.npz")
    doc = json.loads(str(g["doc"]))
    md = doc["model"]
    m = O.build_toy_model(md["d_model"], md["heads"], md["layers"], seed=md["seed"])
    np.testing.assert_array_equal(m.emb, g["embedding"])
    ctx, qry = O.experiment_tokens(doc["seed"], doc["sequence_len"], doc["query_len"])
    assert ctx == list(g["context_tokens"]) and qry == list(g["query_tokens"])
    plan = O.plan_blocks(doc["sequence_len"], doc["block_size"], doc["hosts"])
    spec = O.Anchor(**doc["anchor"])
    lg, sess = O.start_session(m, ctx + qry, plan, spec, O.OraclePrng(doc["seed"] ^ O.ANCHOR_SALT))
    return g, doc, m, lg, sess


@pytest.mark.parametrize("name", SMALL + TINY + ANCHOR)
def test_model_end_to_end(golden_dir, name):
    g, doc, m, lg, sess = _run_case(golden_dir, name)
    np.testing.assert_allclose(lg, g["query_logits"], rtol=1e-4, atol=1e-5)
    toks = O.decode(sess, doc["n_generate"])
    assert toks == list(g["generated"])
    assert O.ledger_csv(sess.ledger) == str(g["ledger_csv"])
    # golden host state is captured after decode (query host holds query + generated rows)
    for hi, host in enumerate(sess.hosts):
        # per-host channel positions, bit-exact (Host.channels[c].positions)
        assert host.pos[0] == list(g[f"host{hi}_pos_ch0"])
        assert host.pos[-1] == list(g[f"host{hi}_pos_last"])
        assert host.role == str(g[f"host{hi}_role"])
        if f"host{hi}_k_ch0" in g:
            np.testing.assert_allclose(host.K[0], g[f"host{hi}_k_ch0"], rtol=1e-5, atol=1e-6)
            np.testing.assert_allclose(host.V[0], g[f"host{hi}_v_ch0"], rtol=1e-5, atol=1e-6)
    if "global_query_logits" in g and plan_n(doc) <= 2:
        # star == global when n <= 2
        np.testing.assert_allclose(g["query_logits"], g["global_query_logits"], rtol=1e-4, atol=1e-5)


def plan_n(doc):
    return -(-doc["sequence_len"] // doc["block_size"])
