"""Where the time of the fused phase-2 exchange goes (one GPU, self-loop boxes).

Graph-replayed variants over a rank's paged cache of --rows rows (Llama-8B heads):
  k2        plain K2 (split fix-up in-kernel), the N = 1 decode
  k2push    K2 whose epilogue pushes into the box (no merge: flags re-raised each time)
  push      exchange_push of a resident partial (no K2)
  push+k3x  exchange_push + K3x merge (one exchange)
  k2push+k3x  K2 push + K3x (two launches)
  exchange(fused)  star_phase2_exchange: partial + push + merge in one K2 launch
  --world W boxes in one process: rank 0's K2 pushes to W boxes (W-1 of them unused).
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_17116_b200 import dist as D  # noqa: E402
from paper_2411_17116_b200 import ops  # noqa: E402


def graph_us(fn, dev, n=200, reps=1):
    fn()
    torch.cuda.synchronize(dev)
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream(dev).wait_stream(s)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        g.replay()
    b.record()
    torch.cuda.synchronize(dev)
    return a.elapsed_time(b) / (n * reps) * 1e3


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rows", type=int, nargs="+", default=[16384, 131072])
    p.add_argument("--splits", type=int, default=0)
    args = p.parse_args()
    dev = torch.device("cuda", 0)
    hq, hkv, d, ps = 32, 8, 128, 128
    for rows in args.rows:
        pages = rows // ps
        kp = ops.prng_fill((pages, hkv, ps, d), 2, 1, 1.0, torch.bfloat16, dev)
        vp = ops.prng_fill((pages, hkv, ps, d), 3, 1, 1.0, torch.bfloat16, dev)
        table = torch.arange(pages, dtype=torch.int32, device=dev).view(1, -1)
        kv_len = torch.tensor([rows], dtype=torch.int32, device=dev)
        q = ops.prng_fill((1, 1, hq, d), 4, 1, 1.0, torch.bfloat16, dev)
        ws = ops.Phase2Workspace()
        ex = D.local_peer_exchanges(1, hq, hkv, d, dev)[0]
        o = torch.zeros(hq, d, device=dev)
        l = torch.zeros(hq, device=dev)
        res = {}
        res["k2"] = graph_us(lambda: ops.phase2_partial(q, kp, vp, table, kv_len, rows,
                                                        n_splits=args.splits, workspace=ws),
                             dev, reps=10)
        res["k2push"] = graph_us(lambda: ex.push_partial(q, kp, vp, table, kv_len, rows,
                                                         n_splits=args.splits, workspace=ws),
                                 dev, reps=10)
        res["exchange(fused)"] = graph_us(
            lambda: ex.exchange(q, kp, vp, table, kv_len, rows, n_splits=args.splits,
                                workspace=ws), dev, reps=10)
        res["push"] = graph_us(lambda: ex.push(o, l, 1, 1, hq, hkv), dev, reps=10)

        def push_merge():
            ex.push(o, l, 1, 1, hq, hkv)
            ex.merge(1, 1, hq, hkv)
        res["push+k3x"] = graph_us(push_merge, dev, reps=10)

        def step():
            ex.push_partial(q, kp, vp, table, kv_len, rows, n_splits=args.splits, workspace=ws)
            return ex.merge(1, 1, hq, hkv)
        res["k2push+k3x"] = graph_us(step, dev, reps=10)
        res["merge_packed(1 part)"] = graph_us(
            lambda: ops.merge_packed(torch.zeros(1, hq * (d + 1), device=dev), hq, d), dev, reps=10)
        print(rows, {k: round(v, 2) for k, v in res.items()}, flush=True)


if __name__ == "__main__":
    main()
