"""K2 in query-encode shape (l_q query rows with the own-tail mask) vs decode, cfg2 heads."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("STAR_LIB_PATH"):  # A/B against another build
    from paper_2411_17116_b200 import _lib  # noqa: E402
    _lib.LIB_PATH = os.environ["STAR_LIB_PATH"]
from paper_2411_17116_b200 import ops  # noqa: E402

dev = torch.device("cuda", 0)
hq, hkv, d, ps = int(os.environ.get('QB_HQ', 32)), 8, 128, 128
for rows in [int(x) for x in os.environ.get("QB_ROWS", "16384,131072").split(",")]:
    pages = rows // ps
    kp = ops.prng_fill((pages, hkv, ps, d), 2, 1, 1.0, torch.bfloat16, dev)
    vp = ops.prng_fill((pages, hkv, ps, d), 3, 1, 1.0, torch.bfloat16, dev)
    table = torch.arange(pages, dtype=torch.int32, device=dev).view(1, -1)
    kv_len = torch.tensor([rows], dtype=torch.int32, device=dev)
    for lq in [int(x) for x in os.environ.get("QB_LQ", "1,4,16,32").split(",")]:
        q = ops.prng_fill((1, lq, hq, d), 4, 1, 1.0, torch.bfloat16, dev)
        ws = ops.Phase2Workspace()
        ns = int(os.environ.get("QB_SPLITS", "0"))  # 0: the library's choice
        f = lambda: ops.phase2_partial(q, kp, vp, table, kv_len, rows, own_tail=lq, workspace=ws,  # noqa
                                       n_splits=ns)
        f()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(10):
                    f()
        torch.cuda.current_stream().wait_stream(s)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 100 * 1e3
        gbs = rows * hkv * d * 4 / us / 1e3
        print(f"rows={rows} lq={lq} us={us:.1f} GB/s={gbs:.0f}", flush=True)
