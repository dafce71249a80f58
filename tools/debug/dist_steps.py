"""Debug: per-step logit error of decode_dist vs the reference's step_logits (gloo, 2 ranks
on cuda:0).  usage: python tools/debug/dist_steps.py NAME TRANSPORT [graph]"""
import json
import os
import socket
import sys

import numpy as np
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def worker(rank, port, name, transport, world, graph):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2411_17116_b200 as S
    from paper_2411_17116_b200 import dist as D
    torch.backends.cuda.matmul.allow_tf32 = False
    S.set_default_dtype("float32")
    g = np.load(os.path.join(ROOT, "tests", "golden", f"model_{name}.npz"))
    doc = json.loads(str(g["doc"]))
    md = doc["model"]
    w = S.init_model(S.ModelConfig(d_model=md["d_model"], heads=md["heads"], layers=md["layers"], seed=md["seed"]))
    plan = S.partition(doc["sequence_len"], doc["block_size"], doc["hosts"])
    spec = S.AnchorSpec(**doc["anchor"])
    toks = list(g["context_tokens"]) + list(g["query_tokens"])
    logits, sess = D.start_session_dist(w, toks, plan, spec, prng=S.Prng(doc["seed"] ^ 0xA17C4B10C4ED5EED), transport=transport)
    print(rank, "query err", float(np.abs(logits.cpu().numpy() - g["query_logits"]).max()), flush=True)
    for i in range(doc["n_generate"]):
        t = D.decode_dist(sess, 1, graph=graph)
        err = float(np.abs(sess.last_logits.cpu().numpy() - g["step_logits"][i + 1]).max())
        print(rank, "step", i, "tok", t, "ref", int(g["generated"][i]), "err", err,
              "rows", sess.pool.rows(0), sess.pool.kv_len_dev.tolist(), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    name, transport = sys.argv[1], sys.argv[2]
    graph = (sys.argv[3] == "1") if len(sys.argv) > 3 else None
    g = np.load(os.path.join(ROOT, "tests", "golden", f"model_{name}.npz"))
    world = int(json.loads(str(g["doc"]))["hosts"])
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    mp.start_processes(worker, args=(port, name, transport, world, graph), nprocs=world, start_method="spawn")
