"""Multi-rank host logic on CPU: world_size 2 over gloo (no GPU).

The device kernels are replaced by the CPU oracle here ONLY as the checker's
compute stand-in; what is under test is the distributed orchestration of
paper_2411_17116_b200.dist: the per-rank phase-1 shard (blocks, cache rows,
position ids), the all-gather of (out, lse) partials, the ascending-rank merge
and the ledger rows — against the reference's goldens.
"""

import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import star_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_merge(outs, lses):
    o, l = O.merge_partials([x.double().numpy() for x in outs],
                            [x.double().numpy() for x in lses])
    return torch.from_numpy(np.asarray(o)), torch.from_numpy(np.asarray(l))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_17116_b200 import dist as D
        import paper_2411_17116_b200 as S

        res = {}
        # --- phase-1 shard of the small_n5h2 golden (L=70, b=16, a=8, 2 hosts) ---
        g = np.load(os.path.join(GOLDEN, "model_small_n5h2.npz"))
        doc = json.loads(str(g["doc"]))
        plan = S.partition(doc["sequence_len"], doc["block_size"], doc["hosts"])
        spec = S.AnchorSpec(anchor_len=doc["anchor"]["anchor_len"])
        blocks = S.augment(plan, list(g["context_tokens"]), spec, S.Prng(doc["seed"] ^ O.ANCHOR_SALT))
        sh = D.rank_shard(plan, blocks, rank)
        ref_pos = [int(p) for p in g[f"host{rank}_pos_ch0"] if p < doc["sequence_len"]]
        res["shard_positions_ok"] = list(sh.cache_positions) == ref_pos
        res["blocks"] = list(sh.blocks)
        res["seg_ok"] = sh.rows == sum(len(blocks[b].token_ids) for b in sh.blocks)

        # --- gather + ordered merge == attention over the union of the shards ---
        rng = np.random.default_rng(7)
        d, lq = 16, 3
        qm = rng.uniform(-1, 1, (lq, d))
        ks = [rng.uniform(-1, 1, (n, d)) for n in (11, 29)]
        vs = [rng.uniform(-1, 1, (n, d)) for n in (11, 29)]
        o, l = O.partial_attention(qm, ks[rank], vs[rank])
        mo, ml = D.gather_merge(torch.from_numpy(o).float(), torch.from_numpy(l).float(),
                                merge_fn=_oracle_merge)
        fo, fl = O.partial_attention(qm, np.concatenate(ks), np.concatenate(vs))
        res["merge_err"] = float(np.abs(mo.numpy() - fo).max())
        res["lse_err"] = float(np.abs(ml.numpy() - fl).max())
        # an empty rank contributes lse = -inf and is skipped
        if rank == 0:
            o0, l0 = torch.zeros(lq, d), torch.full((lq,), float("-inf"))
        else:
            o0, l0 = torch.from_numpy(o).float(), torch.from_numpy(l).float()
        eo, _ = D.gather_merge(o0, l0, merge_fn=_oracle_merge)
        res["empty_rank_err"] = float(np.abs(eo.numpy() - o).max()) if rank == 1 else 0.0

        # --- ledger rows of one phase-2 step match the reference's closed form ---
        rows = D.phase2_ledger_rows(1, [0, 1], layers=2, heads=2, l_q=4, d=16)
        res["ledger_total"] = sum(r[4] for r in rows)
        res["ledger_head"] = rows[:2]
        q.put((rank, res))
    except Exception as e:  # surface worker failures instead of timing out
        q.put((rank, {"error": repr(e)}))
        raise
    finally:
        dist.destroy_process_group()


def test_world2_gloo_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        res = out[r]
        assert "error" not in res, res
        assert res["shard_positions_ok"], r
        assert res["seg_ok"]
        # partials travel as fp32 (the wire format), the reference merge is fp64
        assert res["merge_err"] < 1e-6 and res["lse_err"] < 1e-6
        assert res["empty_rank_err"] < 1e-6
        # (H-1) * l_q * (d+1) * heads * layers
        assert res["ledger_total"] == 1 * 4 * 17 * 2 * 2
        assert res["ledger_head"] == [(2, 0, 1, "partial_out", 64), (2, 0, 1, "partial_lse", 4)]
    assert out[0]["blocks"] == [0, 1, 2] and out[1]["blocks"] == [3, 4]  # min(i*H//n, H-1)


def test_phase2_ledger_matches_golden_csv():
    """phase2_ledger_rows reproduces the reference ledger of a whole tiny-config session."""
    from paper_2411_17116_b200 import dist as D

    g = np.load(os.path.join(GOLDEN, "model_tiny_s4.npz"))
    doc = json.loads(str(g["doc"]))
    H, layers, hd = doc["model"]["heads"], doc["model"]["layers"], 64
    qh, hosts = doc["hosts"] - 1, list(range(doc["hosts"]))
    rows = [(2, qh, r, "query_broadcast", doc["query_len"]) for r in hosts if r != qh]
    rows += D.phase2_ledger_rows(qh, hosts, layers, H, doc["query_len"], hd)
    for _ in range(doc["n_generate"]):
        rows += [(2, qh, r, "query_broadcast", 1) for r in hosts if r != qh]
        rows += D.phase2_ledger_rows(qh, hosts, layers, H, 1, hd)
    csv = "phase,src,dst,kind,scalar_count\n" + "".join(f"{a},{b},{c},{k},{n}\n" for a, b, c, k, n in rows)
    assert csv == str(g["ledger_csv"])


def _fallback_worker(rank, world, port, failing, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_17116_b200 import dist as D
        from paper_2411_17116_b200 import ops

        # host-only stand-ins: no device here, so the box is a CPU tensor, the IPC export
        # fails on the `failing` rank and "maps" (returns a fake address) elsewhere
        torch.cuda.synchronize = lambda *a, **k: None

        def get_handle(t):
            if rank == failing:
                raise RuntimeError("no CUDA IPC for this allocation")
            return b"\0" * 64, 0

        ops.ipc_get_handle = get_handle
        ops.ipc_open_handle = lambda h, o: 0x1000
        ops.ipc_close_handle = lambda p, o: None
        try:
            D.open_peer_exchange(8, 2, 64, "cpu")
            q.put((rank, "opened"))
        except D.PeerExchangeUnavailable as exc:
            q.put((rank, f"unavailable: {exc}"))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, f"error: {exc!r}"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("failing", [-1, 1])
def test_peer_exchange_setup_outcome_is_collective(failing):
    """open_peer_exchange: one rank unable to export its box makes EVERY rank raise
    PeerExchangeUnavailable (the status is all-gathered), so the transport=auto fallback is
    taken together; with no failure every rank opens."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fallback_worker, args=(r, 2, port, failing, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    if failing < 0:
        assert out == {0: "opened", 1: "opened"}, out
    else:
        assert all(v.startswith("unavailable") and "rank 1" in v for v in out.values()), out
