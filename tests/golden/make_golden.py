"""Generate the golden vectors that pin the oracle (and, through it, the CUDA path).

Runs the UNMODIFIED reference (`starsim` 0.1.0, pure Python/numpy) imported
from /root/reference/pkg/src in the build container, and writes small
fixtures under tests/golden/.  The reference does not travel to the GPU box;
these fixtures do.  Regenerate with:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture names the reference entry point that produced it:
  prng.npz       numerics.Prng / prng_fill          (ss/numerics.py:199-263)
  rope.npz       numerics.rope_apply                (ss/numerics.py:161-180)
  attention.npz  attention.causal_attention / partial_attention /
                 merge_partials / streaming_causal_attention (ss/attention.py:109-210)
  blocking.json  blocking.partition / augment       (ss/blocking.py:49-236)
  model_*.npz    sim.start_session + sim.decode on seeded toy models
                 (ss/sim.py:126-368, ss/toy_model.py:93-196, ss/cli.py:108-228);
                 model_anc_*.npz: the same under every non-default anchor mode
                 (ss/blocking.py:182-236)
  encode_block.npz  blocking.encode_block          (ss/blocking.py:239-265)

`python tests/golden/make_golden.py NAME...` regenerates only the named fixtures
(prng rope attention blocking encode_block model_<case>).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import starsim  # noqa: E402
from starsim import cli  # noqa: E402
from starsim.numerics import Prng, Tensor2D, precision, prng_fill, rope_apply, RopeConfig  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def gen_prng():
    out = {}
    seeds = [0, 1, 7, 0xA17C4B10C4ED5EED, (1 << 64) - 1]
    out["seeds"] = np.array(seeds, dtype=np.uint64)
    out["u64"] = np.array(
        [[Prng(s).next_u64() if i == 0 else 0 for i in range(1)] for s in seeds], dtype=np.uint64
    )
    draws = []
    for s in seeds:
        p = Prng(s)
        draws.append([p.next_u64() for _ in range(64)])
    out["u64"] = np.array(draws, dtype=np.uint64)
    floats = []
    for s in seeds:
        p = Prng(s)
        floats.append([p.next_float() for _ in range(16)])
    out["floats"] = np.array(floats, dtype=np.float64)
    fills32, fills64 = [], []
    for s in seeds:
        with precision("float32"):
            fills32.append(prng_fill(Prng(s), 7, 5, 0.25).a)
        with precision("float64"):
            fills64.append(prng_fill(Prng(s), 7, 5, 0.25).a)
    out["fill32"] = np.stack(fills32)
    out["fill64"] = np.stack(fills64)
    # draws after a partial consumption stay on the same counter stream
    p = Prng(3)
    p.next_u64()
    p.next_u64()
    with precision("float32"):
        out["fill_after2"] = prng_fill(p, 3, 4, 1.0).a
    p = Prng(11)
    out["randint256"] = np.array([p.randint_below(256) for _ in range(200)], dtype=np.int64)
    p = Prng(12)
    out["sample_sorted_100_10"] = np.array(p.sample_sorted(100, 10), dtype=np.int64)
    p = Prng(13)
    out["shuffle_20"] = np.array(p.shuffle(list(range(20))), dtype=np.int64)
    np.savez(os.path.join(HERE, "prng.npz"), **out)


def gen_rope():
    rng = np.random.default_rng(5)
    out = {}
    for name, rows, d, dtype, theta in (
        ("a", 9, 8, np.float32, 10000.0),
        ("b", 33, 64, np.float32, 10000.0),
        ("c", 17, 128, np.float64, 500000.0),
    ):
        x = rng.standard_normal((rows, d)).astype(dtype)
        pos = np.sort(rng.choice(1 << 20, rows, replace=False)).astype(np.int64)
        pos[0] = 0
        with precision(dtype):
            y = rope_apply(Tensor2D(x), pos, RopeConfig(d, theta)).a
        out[f"{name}_x"], out[f"{name}_pos"], out[f"{name}_y"] = x, pos, y
        out[f"{name}_theta"] = np.array(theta)
    np.savez(os.path.join(HERE, "rope.npz"), **out)


def gen_attention():
    from starsim import attention as A

    rng = np.random.default_rng(7)
    out = {}
    cases = [
        ("c0", 6, 6, 4, 0),
        ("c1", 37, 37, 16, 0),
        ("c2", 5, 20, 8, 15),
        ("c3", 64, 64, 64, 0),
    ]
    for name, lq, lk, d, off in cases:
        q = rng.uniform(-1, 1, (lq, d)).astype(np.float32)
        k = rng.uniform(-1, 1, (lk, d)).astype(np.float32)
        v = rng.uniform(-1, 1, (lk, d)).astype(np.float32)
        o = A.causal_attention(Tensor2D(q), Tensor2D(k), Tensor2D(v), q_offset=off).a
        s3 = A.streaming_causal_attention(Tensor2D(q), Tensor2D(k), Tensor2D(v), 3, q_offset=off).a
        pc = A.partial_attention(Tensor2D(q), Tensor2D(k), Tensor2D(v), "causal", q_offset=off)
        pf = A.partial_attention(Tensor2D(q), Tensor2D(k), Tensor2D(v), "full")
        for key, val in (("q", q), ("k", k), ("v", v), ("out", o), ("stream3", s3),
                         ("pc_out", pc.out.a), ("pc_lse", pc.lse),
                         ("pf_out", pf.out.a), ("pf_lse", pf.lse)):
            out[f"{name}_{key}"] = val
        out[f"{name}_off"] = np.array(off)
    # explicit tail mask exactly as sim._gather_merge builds it (ss/sim.py:195-200)
    lq, lk, d = 4, 11, 8
    q = rng.uniform(-1, 1, (lq, d)).astype(np.float32)
    k = rng.uniform(-1, 1, (lk, d)).astype(np.float32)
    v = rng.uniform(-1, 1, (lk, d)).astype(np.float32)
    keep = np.ones((lq, lk), dtype=bool)
    keep[:, lk - lq:] = np.arange(lq)[None, :] <= np.arange(lq)[:, None]
    pm = A.partial_attention(Tensor2D(q), Tensor2D(k), Tensor2D(v), keep)
    out.update(tail_q=q, tail_k=k, tail_v=v, tail_keep=keep, tail_out=pm.out.a, tail_lse=pm.lse)
    # merge of 4 shards vs the concatenation
    lq, lk, d = 3, 40, 16
    q = rng.uniform(-1, 1, (lq, d)).astype(np.float32)
    k = rng.uniform(-1, 1, (lk, d)).astype(np.float32)
    v = rng.uniform(-1, 1, (lk, d)).astype(np.float32)
    cuts = [0, 7, 19, 30, 40]
    parts = [A.partial_attention(Tensor2D(q), Tensor2D(k[a:b]), Tensor2D(v[a:b]), "full")
             for a, b in zip(cuts[:-1], cuts[1:])]
    m = A.merge_partials(parts)
    out.update(merge_q=q, merge_k=k, merge_v=v, merge_cuts=np.array(cuts),
               merge_outs=np.stack([p.out.a for p in parts]),
               merge_lses=np.stack([p.lse for p in parts]),
               merge_out=m.out.a, merge_lse=m.lse)
    np.savez(os.path.join(HERE, "attention.npz"), **out)


def gen_blocking():
    from starsim.blocking import AnchorSpec, augment, partition

    doc = {"partition": [], "augment": []}
    for L, b, H, idle in ((10, 4, None, False), (8, 8, None, False), (131072, 16384, 8, False),
                          (131072, 16384, 4, False), (131072, 16384, 2, False),
                          (131072, 16384, 1, False), (4096, 1024, 4, False),
                          (1048576, 131072, 8, False), (262144, 32768, 8, False),
                          (100, 7, 5, False), (20, 6, 6, True), (1, 1, None, False)):
        p = partition(L, b, H, allow_idle=idle)
        doc["partition"].append({
            "L": L, "b": b, "H": H, "allow_idle": idle, "num_blocks": p.num_blocks,
            "num_hosts": p.num_hosts, "assignment": list(p.host_assignment),
            "spans": [list(p.block_span(i)) for i in range(p.num_blocks)],
        })
    rng = np.random.default_rng(3)
    tokens = [int(t) for t in rng.integers(0, 256, 23)]
    for content in starsim.blocking.CONTENT_MODES:
        for position in starsim.blocking.POSITION_MODES:
            for a_len in (None, 3, 6):
                plan = partition(23, 6, 2)
                spec = AnchorSpec(content, position, a_len, constant_token_id=9, token_range=50)
                blocks = augment(plan, tokens, spec, Prng(99))
                doc["augment"].append({
                    "L": 23, "b": 6, "H": 2, "content_mode": content, "position_mode": position,
                    "anchor_len": a_len, "constant_token_id": 9, "token_range": 50, "prng_seed": 99,
                    "tokens": tokens,
                    "blocks": [{"token_ids": list(bl.token_ids), "position_ids": list(bl.position_ids),
                                "anchor_prefix_len": bl.anchor_prefix_len,
                                "block_index": bl.block_index} for bl in blocks],
                })
    # star_model pair counts (ss/baselines.py:124-160)
    doc["star_model"] = []
    for L, b, a, d, heads, lq, ng, H in ((16, 4, None, 8, 1, 0, 0, None),
                                         (131072, 16384, 16384, 128, 32, 1, 0, 8),
                                         (4096, 1024, 1024, 64, 4, 32, 16, 4),
                                         (1048576, 131072, 131072, 128, 32, 1, 64, 8),
                                         (262144, 32768, 32768, 128, 64, 1, 0, 8)):
        r = starsim.star_model(L, b, a, d, heads, lq, ng, H)
        doc["star_model"].append({"args": [L, b, a, d, heads, lq, ng, H], **r.to_json()})
    with open(os.path.join(HERE, "blocking.json"), "w") as f:
        json.dump(doc, f, indent=1, sort_keys=True)


MODEL_CASES = {
    # cfg1 (BASELINE.json configs[0]): 2 layers, 4 heads x 64, 4K ctx, b = a = 1K, 4 hosts,
    # 32-token query + 16 greedy tokens, fp32.  Model seeds {0,4,7}; the token/anchor seed is
    # the CLI default 0 (ss/cli.py:145) -- seeds 4 and 7 then emit non-degenerate token streams.
    "tiny_s0": dict(d_model=256, heads=4, layers=2, seed=0, L=4096, b=1024, a=1024, H=4, lq=32, ng=16),
    "tiny_s4": dict(d_model=256, heads=4, layers=2, seed=4, L=4096, b=1024, a=1024, H=4, lq=32, ng=16),
    "tiny_s7": dict(d_model=256, heads=4, layers=2, seed=7, L=4096, b=1024, a=1024, H=4, lq=32, ng=16),
    # small cases: exact regime (n <= 2), multi-block-per-host, ragged last block
    "small_n2": dict(d_model=32, heads=2, layers=2, seed=1, L=64, b=32, a=32, H=2, lq=5, ng=6),
    "small_n5h2": dict(d_model=32, heads=2, layers=2, seed=2, L=70, b=16, a=8, H=2, lq=4, ng=5),
    "small_n4h4": dict(d_model=48, heads=3, layers=1, seed=3, L=40, b=10, a=10, H=4, lq=3, ng=4),
}


# every non-default anchor mode through the whole protocol (phase 1 anchors -> caches ->
# phase 2 -> greedy tokens): 4 hosts, one block each, b = 64, a = 32
_ANC = dict(d_model=64, heads=2, layers=2, L=256, b=64, a=32, H=4, lq=6, ng=8)
for _name, _cm, _pm, _seed in (("anc_prev", "previous_block", "previous_block", 11),
                               ("anc_randpos", "first_block", "random_sampled", 12),
                               ("anc_prevpos", "first_block", "previous_block", 13),
                               ("anc_shuffled", "shuffled_first_block", "first_block", 14),
                               ("anc_randtok", "random_tokens", "first_block", 15),
                               ("anc_const", "constant_token", "first_block", 16),
                               ("anc_none", "none", "first_block", 17)):
    MODEL_CASES[_name] = dict(_ANC, seed=_seed,
                              anchor={"anchor_len": _ANC["a"], "content_mode": _cm,
                                      "position_mode": _pm, "constant_token_id": 7,
                                      "token_range": 256})


def gen_encode_block():
    """encode_block over every augmented block of a small plan (first-block anchors and the
    previous-block mode), fp32: the own-row K/V cache and its positions."""
    from starsim.blocking import AnchorSpec, augment, encode_block, partition

    rng = np.random.default_rng(21)
    d_model, hd = 32, 16
    out = {}
    with precision("float32"):
        emb = Tensor2D(rng.uniform(-1, 1, (256, d_model)).astype(np.float32))
        wq, wk, wv = (Tensor2D(rng.uniform(-0.3, 0.3, (d_model, hd)).astype(np.float32))
                      for _ in range(3))
        tokens = [int(t) for t in rng.integers(0, 256, 50)]
        for mode in ("first_block", "previous_block"):
            plan = partition(50, 16, 2)
            spec = AnchorSpec(mode, mode, 8)
            blocks = augment(plan, tokens, spec, Prng(5))
            for bl in blocks:
                c = encode_block(bl, emb, wq, wk, wv, RopeConfig(hd, 10000.0), host=1)
                key = f"{mode}_{bl.block_index}"
                out[f"{key}_token_ids"] = np.array(bl.token_ids, dtype=np.int64)
                out[f"{key}_position_ids"] = np.array(bl.position_ids, dtype=np.int64)
                out[f"{key}_anchor"] = np.array(bl.anchor_prefix_len)
                out[f"{key}_k"], out[f"{key}_v"] = c.keys.a, c.values.a
                out[f"{key}_pos"] = np.array(c.positions, dtype=np.int64)
            out[f"{mode}_n"] = np.array(len(blocks))
        out["embedding"], out["wq"], out["wk"], out["wv"] = emb.a, wq.a, wk.a, wv.a
    np.savez(os.path.join(HERE, "encode_block.npz"), **out)


def run_model_case(name, c, with_global=False):
    doc = {
        "model": {"d_model": c["d_model"], "heads": c["heads"], "layers": c["layers"], "seed": c["seed"]},
        "sequence_len": c["L"], "block_size": c["b"],
        "anchor": c.get("anchor", {"anchor_len": c["a"]}),
        "hosts": c["H"], "query_len": c["lq"], "n_generate": c["ng"], "seed": c.get("data_seed", 0),
    }
    cfg = cli.build_experiment(doc)
    w = starsim.init_model(cfg.model)
    plan = starsim.partition(cfg.sequence_len, cfg.block_size, cfg.hosts)
    tokens = cfg.context_tokens + cfg.query_tokens
    logits, sess = starsim.start_session(
        w, tokens, plan, cfg.anchor, prng=Prng(cfg.seed ^ cli._ANCHOR_SALT)
    )
    margins = []
    last = [sess.last_logits.copy()]
    gen = []
    for _ in range(cfg.n_generate):
        srt = np.sort(sess.last_logits)[::-1]
        margins.append(float(srt[0] - srt[1]))
        gen += starsim.decode(sess, 1)
        last.append(sess.last_logits.copy())
    out = {
        "doc": np.array(json.dumps(doc)),
        "context_tokens": np.array(cfg.context_tokens, dtype=np.int64),
        "query_tokens": np.array(cfg.query_tokens, dtype=np.int64),
        "query_logits": logits.a,
        "step_logits": np.stack(last),
        "generated": np.array(gen, dtype=np.int64),
        "margins": np.array(margins),
        "ledger_csv": np.array(sess.ledger.to_csv()),
        "embedding": w.embedding.a,
    }
    for hi, host in enumerate(sess.hosts):
        # channel positions are identical across (layer, head) channels; keep channel 0 and
        # the last one to prove it
        out[f"host{hi}_pos_ch0"] = np.array(host.channels[0].positions, dtype=np.int64)
        out[f"host{hi}_pos_last"] = np.array(host.channels[-1].positions, dtype=np.int64)
        out[f"host{hi}_role"] = np.array(host.role)
        if c["d_model"] <= 64:
            out[f"host{hi}_k_ch0"] = host.channels[0].keys.a
            out[f"host{hi}_v_ch0"] = host.channels[0].values.a
    if with_global:
        gl = starsim.forward_global(w, tokens)
        out["global_query_logits"] = gl.a[cfg.sequence_len:]
    np.savez_compressed(os.path.join(HERE, f"model_{name}.npz"), **out)
    return gen, margins


def main(names=None):
    gens = {"prng": gen_prng, "rope": gen_rope, "attention": gen_attention,
            "blocking": gen_blocking, "encode_block": gen_encode_block}
    for key, fn in gens.items():
        if not names or key in names:
            fn()
    for name, c in MODEL_CASES.items():
        if names and f"model_{name}" not in names:
            continue
        gen, margins = run_model_case(name, c, with_global=c["L"] <= 128)
        print(name, gen, "min margin %.3g" % min(margins))


if __name__ == "__main__":
    main(sys.argv[1:])
