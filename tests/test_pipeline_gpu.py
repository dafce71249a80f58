"""Host-buffer phase-1 pipeline (paper_2411_17116_b200.pipeline) on the B200.

Both host layouts — augmented (anchor rows repeated per block, ss/blocking.py:206-236)
and context (each context row once, anchors replicated on the device) — must give the
device-resident path's output bit for bit, and the same paged KV cache.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G,rank,L,b,a", [(1, 0, 1024, 256, 256), (2, 1, 1024, 256, 256),
                                          # ragged last block, anchor shorter than a block
                                          (1, 0, 1000, 256, 128), (3, 2, 1500, 384, 200)])
def test_host_pipeline_layouts_match_device_path(G, rank, L, b, a):
    from paper_2411_17116_b200 import ops, pipeline

    dev = torch.device("cuda", 0)
    hq, hkv, d = 8, 2, 128
    n = -(-L // b)
    pos, seg, own = [], [0], []
    for i in range(n):
        if min(i * G // n, G - 1) != rank:
            continue
        span = list(range(i * b, min(i * b + b, L)))
        rows = list(range(a)) + span if i else span
        pos += rows
        seg.append(seg[-1] + len(rows))
        own.append(len(span))
    R = seg[-1]
    positions = torch.tensor(pos, dtype=torch.int64, device=dev)
    qf, kf, vf = (ops.prng_fill((L, h, d), s, 1, 1.0, torch.bfloat16, dev)
                  for s, h in ((1, hq), (2, hkv), (3, hkv)))
    q, k, v = (t.index_select(0, positions).contiguous() for t in (qf, kf, vf))
    own_rows = sum(own)
    page = 128
    n_pages = -(-own_rows // page) + 1
    table = torch.arange(n_pages, dtype=torch.int32, device=dev)
    cache_rows = torch.full((R,), -1, dtype=torch.int64)
    c0 = 0
    for i, o in enumerate(own):
        cache_rows[seg[i + 1] - o:seg[i + 1]] = torch.arange(c0, c0 + o)
        c0 += o
    cache_rows = cache_rows.to(dev)

    def pools():
        kp = torch.zeros((n_pages, hkv, page, d), dtype=torch.bfloat16, device=dev)
        return kp, torch.zeros_like(kp)

    # device-resident reference path: fused prologue + one K1 launch over all segments
    kp0, vp0 = pools()
    q_rot, k_rot = torch.empty_like(q), torch.empty_like(k)
    ops.rope_qkv(q, k, v, positions, 10000.0, q_out=q_rot, k_out=k_rot, cache_rows=cache_rows,
                 k_pages=kp0, v_pages=vp0, page_table=table)
    ref, _ = ops.phase1_fwd(q_rot, k_rot, v, seg)
    torch.cuda.synchronize()

    plan = pipeline.LayerEncodePlan.create(seg, own, hq, hkv, d, dev)
    pin = lambda t: t.cpu().pin_memory()  # noqa: E731
    out_h = torch.empty((R, hq, d), dtype=torch.bfloat16, pin_memory=True)
    kp1, vp1 = pools()
    pipeline.encode_layer_host(plan, pin(q), pin(k), pin(v), positions, kp1, vp1, table, out_h)
    torch.cuda.synchronize()
    assert torch.equal(out_h.to(dev), ref)
    assert torch.equal(kp1, kp0) and torch.equal(vp1, vp0)

    n_ctx = plan.set_context_layout(np.array(pos))
    uniq = torch.unique(positions)
    assert n_ctx == uniq.numel()
    out_c = torch.zeros((R, hq, d), dtype=torch.bfloat16, pin_memory=True)
    kp2, vp2 = pools()
    pipeline.encode_layer_host_context(plan, pin(qf.index_select(0, uniq)), pin(kf.index_select(0, uniq)),
                                       pin(vf.index_select(0, uniq)), positions, kp2, vp2, table,
                                       out_c)
    torch.cuda.synchronize()
    assert torch.equal(out_c.to(dev), ref)
    assert torch.equal(kp2, kp0) and torch.equal(vp2, vp0)


def test_back_to_back_encodes_without_waiting():
    """Two encodes of different inputs queued back to back with wait=False (the next fill
    overlaps the previous drain): each output equals its own device-path reference."""
    from paper_2411_17116_b200 import ops, pipeline

    dev = torch.device("cuda", 0)
    L, b, a, hq, hkv, d = 1024, 256, 256, 8, 2, 128
    n = L // b
    pos, seg, own = [], [0], []
    for i in range(n):
        rows = list(range(a)) + list(range(i * b, i * b + b)) if i else list(range(b))
        pos += rows
        seg.append(seg[-1] + len(rows))
        own.append(b)
    R = seg[-1]
    positions = torch.tensor(pos, dtype=torch.int64, device=dev)
    page = 128
    n_pages = -(-sum(own) // page) + 1
    table = torch.arange(n_pages, dtype=torch.int32, device=dev)
    kp = torch.zeros((n_pages, hkv, page, d), dtype=torch.bfloat16, device=dev)
    vp = torch.zeros_like(kp)
    plan = pipeline.LayerEncodePlan.create(seg, own, hq, hkv, d, dev)
    refs, outs, hosts = [], [], []
    for seed in (11, 23):
        q, k, v = (ops.prng_fill((L, h, d), seed + s_, 1, 1.0, torch.bfloat16, dev)
                   .index_select(0, positions).contiguous() for s_, h in ((1, hq), (2, hkv), (3, hkv)))
        q_rot, k_rot = torch.empty_like(q), torch.empty_like(k)
        ops.rope(q, positions, 10000.0, out=q_rot)
        ops.rope(k, positions, 10000.0, out=k_rot)
        refs.append(ops.phase1_fwd(q_rot, k_rot, v, seg)[0])
        hosts.append(tuple(t.cpu().pin_memory() for t in (q, k, v)))
        outs.append(torch.empty((R, hq, d), dtype=torch.bfloat16, pin_memory=True))
    torch.cuda.synchronize()
    for (hq_, hk_, hv_), out_h in zip(hosts, outs):
        pipeline.encode_layer_host(plan, hq_, hk_, hv_, positions, kp, vp, table, out_h,
                                   wait=False)
    plan.synchronize()
    for ref, out_h in zip(refs, outs):
        assert torch.equal(out_h.to(dev), ref)
