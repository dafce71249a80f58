"""Benchmark of the Star Attention two-phase hot path on B200.

Workload (BASELINE.json configs[1], the metric's own config): Llama-3.1-8B
attention shapes — 32 q / 8 kv heads, head_dim 128 — over a 128K context cut
into 16K blocks with 16K first-block anchors, bf16, one layer per step.

One step = phase 1 of one layer over the whole context: the fused prologue
(RoPE of Q and K at the augmented position ids + own-row K/V write into the
paged cache, one kernel) and the tcgen05 causal block encode (K1) over every
anchor-augmented block this rank owns (one launch).  `value` = context tokens encoded per second over all ranks (strong
scaling: the 128K context is fixed, blocks are sharded by partition()).
After the timed steps, the per-token phase-2 decode latency (K2 split-KV
partial over the rank's paged cache; at N > 1 its epilogue pushes (out, lse) into
every rank's box over NVLink peer memory and K3x merges) is measured the same way
and reported under "decode".

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "context-encode tokens/s & per-token decode latency (128K ctx), 1–8 B200"
CFG = dict(L=131072, b=16384, a=16384, hq=32, hkv=8, d=128, seed=0)


def bench_config(world):
    """The `config` object of BOTH arms (ours and --impl reference): identical by construction."""
    return {"workload": "cfg2: Llama-3.1-8B attention (32 q / 8 kv heads, head_dim 128), 128K "
                        "context, block 16K, first-block anchor 16K, phase-1 encode of one layer "
                        "per step",
            "context": CFG["L"], "block": CFG["b"], "anchor": CFG["a"], "heads_q": CFG["hq"],
            "heads_kv": CFG["hkv"], "head_dim": CFG["d"],
            "parallelism": f"star{world} (blocks sharded by partition)",
            "l2": "inputs (>= 1.5 GB per rank) exceed the 126 MB L2; no flush needed"}


def star_pairs(L, b, a):
    n = -(-L // b)
    return sum((m := (min(b, L - i * b) + (a if i else 0))) * (m + 1) // 2 for i in range(n))


def rank_blocks(L, b, a, G, rank):
    """(block index, augmented rows m_i, own rows) for the blocks partition() gives `rank`."""
    n = -(-L // b)
    owner = [min(i * G // n, G - 1) for i in range(n)]
    out = []
    for i in range(n):
        if owner[i] == rank:
            own = min(b, L - i * b)
            out.append((i, own + (a if i else 0), own))
    return out


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Clock / throttle-reason sampling during the timed region (B200_PROFILING.md clocks
    line): NVML every 20 ms (nvidia-smi as the fallback, ~5 samples/s)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, {reason names})
        self._stop = threading.Event()
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
        except Exception:
            self._nvml = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        flags = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                 nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        return float(sm), float(mx), {n for n, f in zip(self.NAMES, flags) if bits & f}

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        r = [x.strip() for x in out.split(",")]
        sm = float(r[0]) if r[0].replace(".", "").isdigit() else None
        mx = float(r[1]) if r[1].replace(".", "").isdigit() else None
        return sm, mx, {self.NAMES[i] for i in range(4)
                        if len(r) > 3 + i and r[3 + i].lower().startswith("active")}

    def _run(self):
        while not self._stop.is_set():
            try:
                self.rows.append(self._sample_nvml() if self._nvml else self._sample_smi())
            except Exception:
                pass
            self._stop.wait(0.02 if self._nvml else 0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows if r[0] is not None]
        mx = [r[1] for r in self.rows if r[1] is not None]
        reasons = sorted(set().union(*[r[2] for r in self.rows]))
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml" if self._nvml else "nvidia-smi"}


# ----------------------------------------------------------------------------- CPU legs
def blas_threads():
    """(library, threads) of numpy's BLAS (threadpoolctl), for the cpu_baseline record."""
    try:
        from threadpoolctl import threadpool_info

        info = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        if info:
            return f"{info[0].get('internal_api')} {info[0].get('version')}", int(info[0]["num_threads"])
    except Exception:  # noqa: BLE001 - informational only
        pass
    return "unknown", None


def cpu_unit(rows):
    """Seconds for the oracle's causal_attention (numpy restatement of ss/attention.py:109-122)
    on one (q-head, `rows`-row augmented block) unit, fp32, d = 128, inputs drawn by the
    reference Prng recipe.  Materialises the full rows x rows score matrix as the reference
    does (17.9 GB RSS at 32,768 rows)."""
    from oracle import star_oracle as O

    d = CFG["d"]
    q = O.counter_fill(1, rows * d).astype(np.float32).reshape(rows, d)
    k = O.counter_fill(2, rows * d).astype(np.float32).reshape(rows, d)
    v = O.counter_fill(3, rows * d).astype(np.float32).reshape(rows, d)
    t0 = time.perf_counter()
    O.causal_attention(q, k, v)
    return time.perf_counter() - t0


def cpu_layer_seconds(t_first, t_aug):
    """One cfg2 layer on the CPU = Hq x (block 0's unit + 7 anchor-augmented units): the units
    are independent and identical per (head, block), so this is exact."""
    n = -(-CFG["L"] // CFG["b"])
    return CFG["hq"] * (t_first + (n - 1) * t_aug)


CPU_SAMPLE = ("oracle causal_attention (numpy, fp32) on full-size units: one (q-head, block 0) "
              "unit of 16,384 rows and one (q-head, augmented block) unit of 32,768 rows; "
              "layer time = 32 heads x (t_16K + 7 x t_32K) (units independent and identical, "
              "BASELINE.md §3)")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    b, a = CFG["b"], CFG["a"]
    # warm-up: the block-0 unit (measured once, it enters the layer time) then augmented units
    t_first = cpu_unit(b)
    for _ in range(max(0, args.warmup - 1)):
        cpu_unit(b + a)
    ts = [cpu_unit(b + a) for _ in range(args.steps)]
    t_aug = float(np.median(ts))
    layer_s = cpu_layer_seconds(t_first, t_aug)
    val = CFG["L"] / layer_s
    lib, nthr = blas_threads()
    cores = nthr or os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_aug * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (splitmix64 counter fill)",
        "config": bench_config(args.gpus),
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": cores, "kind": "port",
                         "sample": CPU_SAMPLE, "blas": lib, "blas_threads": nthr,
                         "host_cpus": os.cpu_count(), "t_unit_16k_s": t_first,
                         "t_unit_32k_s": t_aug, "layer_s": layer_s},
        "step_note": "one step = one full-size 32,768-row (q-head, augmented block) unit; "
                     "ms_per_step is that unit's time, value extrapolates it to the layer",
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU leg
def run_ours(args):
    import torch
    import torch.distributed as dist

    if os.environ.get("STAR_BENCH_HANG_DUMP"):  # diagnostics: stack dump + exit if stuck
        import faulthandler

        faulthandler.dump_traceback_later(float(os.environ["STAR_BENCH_HANG_DUMP"]), exit=True)

    from paper_2411_17116_b200 import dist as D
    from paper_2411_17116_b200 import ops
    from paper_2411_17116_b200.numerics import Prng  # noqa: F401  (API import check)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = os.environ.get("STAR_BENCH_BACKEND", "nccl")  # gloo: multi-rank logic test on 1 GPU
    if backend != "nccl":
        local %= torch.cuda.device_count()  # ranks may share a device in this test mode
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg_info = {"backend": None, "world": 1}
    nccl_log = f"/tmp/star_bench_nccl.{os.getpid()}.log"
    if world > 1:
        if backend == "nccl":
            # NCCL's own INIT lines (communicator size, transports) go to a per-process file;
            # rank 0 quotes its communicator lines in the JSON line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", nccl_log)
            dist.init_process_group("nccl", device_id=dev)
            dist.barrier()
        else:
            dist.init_process_group(backend)
        pg_info = {"backend": dist.get_backend(), "world": dist.get_world_size(),
                   "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))
                   if backend == "nccl" else None}
        if backend == "nccl":
            try:
                with open(os.environ["NCCL_DEBUG_FILE"]) as f:
                    pg_info["nccl_init"] = [ln.strip() for ln in f
                                            if "nranks" in ln or "Init COMPLETE" in ln][:8]
            except OSError:
                pg_info["nccl_init"] = None
    G = world
    L, b, a, hq, hkv, d, seed = (CFG[k] for k in ("L", "b", "a", "hq", "hkv", "d", "seed"))
    blocks = rank_blocks(L, b, a, G, rank)
    seg = [0]
    pos_list = []
    for i, m, own in blocks:
        seg.append(seg[-1] + m)
        start = i * b
        pos_list.append(np.concatenate([np.arange(a), np.arange(start, start + own)]) if i
                        else np.arange(start, start + own))
    R = seg[-1]
    positions = torch.from_numpy(np.concatenate(pos_list).astype(np.int64)).to(dev)

    # synthetic pre-RoPE Q/K/V: row r of an augmented block is context row positions[r]
    # (first_block anchors repeat block 0's rows), drawn from splitmix64 counter streams
    def ctx_gather(seed_x, heads):
        full = ops.prng_fill((L, heads, d), seed_x, 1, 1.0, torch.bfloat16, dev)
        return full.index_select(0, positions).contiguous()

    q_raw = ctx_gather(seed ^ 1, hq)
    k_raw = ctx_gather(seed ^ 2, hkv)
    v = ctx_gather(seed ^ 3, hkv)
    q_rot = torch.empty_like(q_raw)
    k_rot = torch.empty_like(k_raw)
    out = torch.empty_like(q_raw)
    own_rows = sum(o for _, _, o in blocks)
    page = 128
    n_pages = -(-own_rows // page) + 1
    kpool = torch.zeros((n_pages, hkv, page, d), dtype=torch.bfloat16, device=dev)
    vpool = torch.zeros_like(kpool)
    table = torch.arange(n_pages, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    launches = [0]

    # anchor dedup applies when this rank holds block 0 and later blocks
    dedup_rows = a if (blocks and blocks[0][0] == 0 and len(blocks) > 1) else 0

    # logical cache row of every augmented row (own rows only; anchors are not cached)
    cache_rows_h = np.full(R, -1, dtype=np.int64)
    row0 = 0
    for (i, m, own), s0 in zip(blocks, seg[:-1]):
        cache_rows_h[s0 + m - own:s0 + m] = np.arange(row0, row0 + own)
        row0 += own
    cache_rows = torch.from_numpy(cache_rows_h).to(dev)

    def step(qr, kr, vv, o, k1_events=None, dedup=0):
        # fused prologue (RoPE q/k + own-row K/V page write), then the K1 block encode
        ops.rope_qkv(qr, kr, vv, positions, 10000.0, q_out=q_rot, k_out=k_rot,
                     cache_rows=cache_rows, k_pages=kpool, v_pages=vpool, page_table=table)
        if k1_events is not None:
            k1_events[0].record(stream)
        ops.phase1_fwd(q_rot, k_rot, vv, seg, out=o, dedup_anchor_rows=dedup)
        if k1_events is not None:
            k1_events[1].record(stream)
        launches[0] += 2

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---------------- device-resident timing (value) ----------------
    for _ in range(args.warmup):
        step(q_raw, k_raw, v, out)
    barrier()
    k1_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
             for _ in range(args.steps)]
    launches[0] = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for s in range(args.steps):
            step(q_raw, k_raw, v, out, k1_ev[s])
        e1.record(stream)
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    k1_local = float(np.mean([x.elapsed_time(y) for x, y in k1_ev]))
    flops_local = sum(m * (m + 1) // 2 for _, m, _ in blocks) * hq * 4 * d
    per_rank = [(k1_local, flops_local)]
    if world > 1:  # every rank's K1 time and work: the roofline names the busiest rank
        t = torch.tensor([k1_local, float(flops_local)], dtype=torch.float64, device=dev)
        allt = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        per_rank = [(float(x[0]), int(x[1])) for x in allt]
    busiest = max(range(world), key=lambda r: per_rank[r][0])
    k1_ms = per_rank[busiest][0]
    gpu_launches = launches[0]
    value = L / (ms * 1e-3)

    # ---------------- secondary: the same step with anchor dedup ----------------
    # (only ranks holding block 0 and later blocks run it; every rank takes the same
    # barriers, so the collectives stay matched)
    dedup_info = None
    if dedup_rows:
        ref_out = out.clone()
        out.fill_(float("nan"))  # every row must be rewritten by the deduplicated launch
        step(q_raw, k_raw, v, out, dedup=dedup_rows)
    barrier()
    if dedup_rows:
        same = torch.equal(out, ref_out)
        del ref_out
        dk = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
    barrier()
    if dedup_rows:
        e0.record(stream)
        for s in range(args.steps):
            step(q_raw, k_raw, v, out, dk[s], dedup=dedup_rows)
        e1.record(stream)
    barrier()
    if dedup_rows:
        dd_ms = e0.elapsed_time(e1) / args.steps
        dd_k1 = float(np.mean([x.elapsed_time(y) for x, y in dk]))
        n_dd = len(blocks) - 1
        flops_dd = (sum(m * (m + 1) // 2 for _, m, _ in blocks) - n_dd * (dedup_rows // 128 * 128)
                    * (dedup_rows // 128 * 128 + 1) // 2) * hq * 4 * d
        dedup_info = {"value": L / (dd_ms * 1e-3), "unit": "tokens/s", "ms_per_step": dd_ms,
                      "kernel_ms": dd_k1, "computed_flops_per_launch": flops_dd,
                      "achieved_tflops_computed": flops_dd / (dd_k1 * 1e-3) / 1e12,
                      "outputs_bit_identical_to_full": bool(same),
                      "note": "SURVEY §8 f3: anchor rows of blocks 1..n-1 repeat block 0's "
                              "computation (first_block anchors); computed once and written to "
                              "every block. Not used for `value`."}

    # ---------------- roofline of K1 (the busiest rank's launch) ----------------
    flops = per_rank[busiest][1]
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    peak_sus = peaks.get("bf16_tflops_sustained", 1400.0)
    peak_burst = peaks.get("bf16_tflops", 1590.0)
    achieved = flops / (k1_ms * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_k1_traffic.json")) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    except OSError:
        pass

    # ---------------- e2e through the host-buffer API ----------------
    # pinned host Q/K/V in, pinned host out; per-block pipeline (H2D || RoPE+K1+KV write ||
    # D2H) through paper_2411_17116_b200.pipeline.encode_layer_host
    e2e = None
    if not args.no_e2e:
        from paper_2411_17116_b200 import pipeline

        hq_raw = torch.empty(q_raw.shape, dtype=q_raw.dtype, pin_memory=True)
        hk_raw = torch.empty(k_raw.shape, dtype=k_raw.dtype, pin_memory=True)
        hv = torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
        hout = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
        hq_raw.copy_(q_raw)
        hk_raw.copy_(k_raw)
        hv.copy_(v)
        plan = pipeline.LayerEncodePlan.create(seg, [o for _, _, o in blocks], hq, hkv, d, dev)

        def e2e_step():
            # back-to-back layers: a call returns without joining the current stream, so the
            # next layer's H2D fill overlaps this layer's D2H drain (per-segment events keep the
            # staging / output buffers ordered, pipeline._encode)
            pipeline.encode_layer_host(plan, hq_raw, hk_raw, hv, positions, kpool, vpool, table,
                                       hout, wait=False)
            launches[0] += 2 * len(blocks)

        def time_e2e(fn):
            for _ in range(max(1, args.warmup // 2)):
                fn()
            stream.wait_event(plan.done)
            barrier()
            x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n_e2e = max(1, min(args.steps, 5))
            x0.record(stream)
            for _ in range(n_e2e):
                fn()
            stream.wait_event(plan.done)  # every step's D2H inside the timed region
            x1.record(stream)
            barrier()
            return max_over_ranks(x0.elapsed_time(x1) / n_e2e)

        aug_ms = time_e2e(e2e_step)
        aug_ok = torch.equal(plan.out, out)
        aug_h2d = int((hq_raw.numel() + hk_raw.numel() + hv.numel()) * 2)
        del hq_raw, hk_raw, hv
        # context layout: each distinct context row crosses PCIe once; block 0's rows are
        # replicated into the anchor slots on the device (first-block anchors)
        n_ctx = plan.set_context_layout(positions.cpu().numpy())
        uniq = torch.unique(positions)
        assert uniq.numel() == n_ctx

        def ctx_host(seed_x, heads):
            full = ops.prng_fill((L, heads, d), seed_x, 1, 1.0, torch.bfloat16, dev)
            h = torch.empty((n_ctx, heads, d), dtype=torch.bfloat16, pin_memory=True)
            h.copy_(full.index_select(0, uniq))
            return h

        cq, ck, cv = ctx_host(seed ^ 1, hq), ctx_host(seed ^ 2, hkv), ctx_host(seed ^ 3, hkv)
        plan.out.zero_()

        def e2e_ctx_step():
            pipeline.encode_layer_host_context(plan, cq, ck, cv, positions, kpool, vpool, table,
                                               hout, wait=False)
            launches[0] += 2 * len(blocks)

        e2e_ms = time_e2e(e2e_ctx_step)
        ok = torch.equal(plan.out, out) and torch.equal(hout.to(dev), out)
        e2e = {"value": L / (e2e_ms * 1e-3), "unit": "tokens/s",
               "h2d_bytes_per_step": int((cq.numel() + ck.numel() + cv.numel()) * 2),
               "d2h_bytes_per_step": int(hout.numel() * 2), "ms_per_step": e2e_ms,
               "matches_device_path": bool(ok),
               "path": "pinned host Q/K/V (context layout: each context row once) -> per-block "
                       "pipeline (H2D | anchor rows replicated on device | star_rope + "
                       "star_phase1_fwd + star_kv_write | D2H of every encoded row) -> pinned "
                       "host out",
               "augmented_layout": {"value": L / (aug_ms * 1e-3), "ms_per_step": aug_ms,
                                    "h2d_bytes_per_step": aug_h2d,
                                    "matches_device_path": bool(aug_ok),
                                    "path": "pinned host Q/K/V with anchor rows repeated per "
                                            "block (the reference's augmented layout)"}}
        del cq, ck, cv, hout, plan

    # ---------------- phase-2 decode latency (B=1, one layer) ----------------
    del q_raw, k_raw, q_rot, out
    torch.cuda.empty_cache()
    qd = ops.prng_fill((1, 1, hq, d), seed ^ 4, 1, 1.0, torch.bfloat16, dev)
    kv_len = torch.tensor([own_rows], dtype=torch.int32, device=dev)
    # Phase-2 exchange across ranks, two transports:
    #  * peer (the product path, star_phase2_exchange): K2's split fix-up stores each slice
    #    of the rank's partial into every rank's box over NVLink peer memory as {value,
    #    epoch} words, then folds every rank's words of the same slice — the whole exchange
    #    in one kernel.  At N = 1 it runs as a self-loop (one box) to measure its overhead
    #    over plain K2.
    #  * collective (for comparison, N > 1): K2 writes (out, lse) into the packed wire
    #    format [hq*d | hq], one NCCL all-gather, K3 merges the gathered parts in place.
    packed, po, pl = ops.packed_partial(hq, d, dev)
    gathered = torch.empty(world * hq * (d + 1), dtype=torch.float32, device=dev)
    ws = ops.Phase2Workspace()
    peer_note = None
    if world > 1:
        try:
            ex = D.open_peer_exchange(hq, hkv, d, dev)
        except D.PeerExchangeUnavailable as exc:  # same outcome on every rank
            ex, peer_note = None, f"peer exchange unavailable ({exc}); all-gather transport"
    else:
        ex = D.local_peer_exchanges(1, hq, hkv, d, dev)[0]

    def k2_only():
        return ops.phase2_partial(qd, kpool, vpool, table.view(1, -1), kv_len, own_rows,
                                  out=po.view(1, 1, hq, d), lse=pl.view(1, 1, hq), workspace=ws)

    def peer_step():
        # one kernel: partial + push to every box + merge of every rank's partial
        return ex.exchange(qd, kpool, vpool, table.view(1, -1), kv_len, own_rows, workspace=ws)

    def collective_step():
        k2_only()
        dist.all_gather_into_tensor(gathered, packed)
        return ops.merge_packed(gathered.view(world, -1), hq, d)

    decode_step = (peer_step if ex is not None else collective_step) if world > 1 else k2_only

    def capture(fn, reps=1):
        """CUDA graph of `reps` calls of fn (a decode loop replays a fixed graph per token)."""
        fn()  # allocate workspaces outside capture
        torch.cuda.synchronize(dev)
        barrier()
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                for _ in range(reps):
                    fn()
        stream.wait_stream(side)
        return g

    def time_replays(g, n, per=1):
        for _ in range(3):
            g.replay()
        barrier()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        for _ in range(n):
            g.replay()
        d1.record(stream)
        barrier()
        return max_over_ranks(d0.elapsed_time(d1) / (n * per) * 1e3)

    # every rank captures and replays the same graphs in the same order (the peer
    # exchange pairs the ranks' k-th exchanges)
    graph = capture(decode_step)
    timing = "CUDA-graph replay; kernel_us = 100 back-to-back K2 launches"
    replay = graph.replay
    n_k2 = 20
    k2_graph = capture(lambda: ops.phase2_partial(qd, kpool, vpool, table.view(1, -1), kv_len,
                                                  own_rows, workspace=ws), n_k2)
    exch_us = time_replays(capture(peer_step), 200) if ex is not None else peer_note
    coll_us = None
    if world > 1 and backend != "nccl":
        coll_us = f"unmeasured ({backend} collectives cannot be graph-captured)"
    elif world > 1:
        try:
            coll_us = time_replays(capture(collective_step), 200)
        except Exception as exc:  # a backend without graph capture
            torch.cuda.synchronize(dev)
            coll_us = f"unmeasured ({type(exc).__name__})"

    dec_us = time_replays(graph, 200)
    k2_us = time_replays(k2_graph, 5, per=n_k2)
    # phase-2 query encode (BASELINE configs[0]'s l_q = 32 query tokens at these heads; the
    # query rank's own-tail mask), informational: K2 over the rank's cache
    lq_enc = 32
    q_enc = ops.prng_fill((1, lq_enc, hq, d), seed ^ 5, 1, 1.0, torch.bfloat16, dev)
    ws_enc = ops.Phase2Workspace()
    enc_graph = capture(lambda: ops.phase2_partial(q_enc, kpool, vpool, table.view(1, -1), kv_len,
                                                   own_rows, own_tail=lq_enc, workspace=ws_enc), 5)
    enc_us = time_replays(enc_graph, 5, per=5)
    kv_bytes = own_rows * hkv * d * 2 * 2
    decode = {
        "us_per_token_per_layer": dec_us, "batch": 1, "context": L,
        "kernel_us": k2_us, "timing": timing,
        "roofline": {"bound": "hbm", "achieved": kv_bytes / (k2_us * 1e-6) / 1e9,
                     "peak": peaks.get("hbm_gbs", 6532.9), "unit": "GB/s",
                     "frac": kv_bytes / (k2_us * 1e-6) / 1e9 / peaks.get("hbm_gbs", 6532.9),
                     "bytes_per_launch": kv_bytes,
                     "note": "K2 split-KV partial + in-GPU split merge; bytes = local KV rows x 8 heads x 128 x 2 (K,V) x 2 B"},
        "exchange": (peer_note or "fused peer exchange, one kernel per token-layer: K2 stores "
                     "its partial into every rank's box over NVLink peer memory and merges "
                     "every rank's partial as the words land (no NCCL)") if world > 1
                    else "none (1 rank: the K2 partial is the answer)",
        "peer_exchange_us": exch_us,
        "peer_exchange_note": ("star_phase2_exchange per token" if world > 1 else
                               "star_phase2_exchange as a one-box self-loop: the fused path's "
                               "overhead over plain K2 at N = 1"),
        "collective_us": coll_us,
        "collective_note": "K2 + NCCL all_gather of packed fp32 (out | lse) + K3, for comparison",
        "query_encode": {"l_q": lq_enc, "us_per_layer": enc_us, "own_tail": lq_enc,
                         "note": "phase-2 query encode: K2 over the rank's cache with the query "
                                 "rank's own-tail causal mask (G*l_q = 128 rows per kv head, "
                                 "bound by the mma.sync rate, not HBM)"},
    }

    # ---------------- a whole 32-layer decode step through the package API ----------------
    # Llama-3.1-8B has 32 layers: one rank's paged caches for all of them (distinct pages per
    # layer, so nothing is L2-resident between layers), and per layer the graph-safe decode
    # attention of paper_2411_17116_b200.decoding.paged_attend: fused RoPE + append of the new
    # token on the query rank (device row counter), K2 over the rank's pages and, at N > 1,
    # the one-kernel peer exchange.  The model's projections / FFN are not part of the path.
    torch.cuda.empty_cache()
    if world > 1 and ex is None and backend != "nccl":
        decode["layers32"] = {"skipped": f"no peer exchange and {backend} collectives cannot be "
                                         "graph-captured"}
    else:
        decode["layers32"] = decode_layers_step(dev, world, rank, own_rows,
                                                ex if world > 1 else None, k2_us, barrier,
                                                max_over_ranks, peaks)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    sweep = None if args.no_sweep else decode_sweep(dev, hq, hkv, d, peaks.get("hbm_gbs", 6532.9))
    shares = None
    cfg1 = None
    if not args.no_sweep and world == 1:
        shares = config_shares(dev, peak_sus)
        cfg1 = cfg1_session(dev)
    cpu = None
    if not args.no_cpu_baseline:
        t_first, t_aug = cpu_unit(b), cpu_unit(b + a)
        lib, nthr = blas_threads()
        cpu = {"value": L / cpu_layer_seconds(t_first, t_aug), "unit": "tokens/s",
               "cores": nthr or os.cpu_count(), "kind": "port", "sample": CPU_SAMPLE,
               "blas": lib, "blas_threads": nthr, "host_cpus": os.cpu_count(),
               "t_unit_16k_s": t_first, "t_unit_32k_s": t_aug}
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (splitmix64 counter fill, reference Prng recipe), random-init shapes",
        "config": bench_config(world),
        "rank0_layout": {"blocks": [i for i, _, _ in blocks], "rows": R},
        "process_group": pg_info,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_sus, "unit": "TFLOP/s",
                     "frac": achieved / peak_sus, "frac_of_burst_peak": achieved / peak_burst,
                     "peak_kind": "measured sustained bf16 (MEASURED_PEAKS.json)",
                     "traffic": traffic, "kernel": "phase1_tc_kernel<128,2>",
                     "flops_per_launch": flops, "kernel_ms": k1_ms, "rank": busiest,
                     "flops_def": "star pairs x Hq x 4 x d (anchor query rows included)",
                     "per_rank": [{"rank": r, "blocks": [i for i, _, _ in rank_blocks(L, b, a, G, r)],
                                   "kernel_ms": t_, "flops": f_,
                                   "tflops": f_ / (t_ * 1e-3) / 1e12 if t_ > 0 else None}
                                  for r, (t_, f_) in enumerate(per_rank)]},
        "decode": decode,
        "decode_sweep": sweep,
        "config_shares": shares,
        "cfg1_session": cfg1,
        "anchor_dedup": dedup_info,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "gpu_launches": gpu_launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def decode_layers_step(dev, world, rank, own_rows, ex, k2_us, barrier, max_over_ranks, peaks,
                       n_layers=32, tokens=32):
    # at N > 1 without a peer exchange the merge is the NCCL all-gather + K3 (captured too)
    """µs per generated token for the attention path of a 32-layer decode step at cfg2, one
    CUDA graph per token, timed over `tokens` replays (max over ranks)."""
    import torch

    from paper_2411_17116_b200 import ops
    from paper_2411_17116_b200.blocking import PagedKVPool
    from paper_2411_17116_b200.decoding import paged_attend

    L, hq, hkv, d = CFG["L"], CFG["hq"], CFG["hkv"], CFG["d"]
    q_rank = world - 1
    room = 128
    pool = PagedKVPool(n_layers, hkv, d, own_rows + room, 128, torch.bfloat16, dev)
    ops.prng_fill(None, 41, out=pool.k.view(-1))
    ops.prng_fill(None, 42, out=pool.v.view(-1))
    pool.layer_rows = [own_rows] * n_layers
    pool.kv_len_dev.fill_(own_rows)
    qn = ops.prng_fill((n_layers, 1, hq, d), 43, 1, 1.0, torch.bfloat16, dev)
    kn = ops.prng_fill((n_layers, 1, hkv, d), 44, 1, 1.0, torch.bfloat16, dev)
    vn = ops.prng_fill((n_layers, 1, hkv, d), 45, 1, 1.0, torch.bfloat16, dev)
    pos = torch.full((1,), L, dtype=torch.int64, device=dev)
    import torch.distributed as tdist

    group = tdist.group.WORLD if (world > 1 and ex is None) else None
    table = ops.DecodeRope(L, room, d, 10000.0, 1, dev)  # cos/sin of the decode positions
    attend = paged_attend(pool, appends=rank == q_rank, max_rows=own_rows + room, theta=10000.0,
                          heads=hq, exchange=ex, group=group, rope_table=table)
    launches = [0]

    finish = getattr(attend, "finish", None)  # fused decode: counters + position, one launch
    if getattr(attend, "prime", None) is not None:
        attend.prime(pos)

    def step():
        for li in range(n_layers):
            attend(li, qn[li], kn[li], vn[li], pos)
        if finish is not None:
            finish(pos)
        else:
            pos.add_(1)

    step()  # eager: workspaces sized before capture
    torch.cuda.synchronize(dev)
    barrier()
    side = torch.cuda.Stream(dev)
    cur = torch.cuda.current_stream(dev)
    side.wait_stream(cur)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
        step()
    cur.wait_stream(side)
    for _ in range(3):
        g.replay()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for _ in range(tokens):
        g.replay()
    e1.record(cur)
    barrier()
    us = max_over_ranks(e0.elapsed_time(e1) / tokens * 1e3)
    kv_bytes = own_rows * hkv * d * 2 * 2
    res = {"layers": n_layers, "us_per_token": us, "us_per_layer": us / n_layers,
           "k2_kernel_us_per_layer": k2_us, "overhead_over_k2": us / n_layers / k2_us - 1.0,
           "hbm_frac_per_layer": kv_bytes / (us / n_layers * 1e-6) / 1e9 / peaks.get("hbm_gbs", 6532.9),
           "tokens_timed": tokens, "cached_rows_per_rank": own_rows,
           "path": ("decoding.paged_attend per layer: " +
                    ("ONE star_phase2_decode launch (RoPE of q in every K2 CTA, the query rank's "
                     "new k/v row written by the K2 CTA that streams it" if finish is not None
                     else "star_kv_append + K2") +
                    (", fused peer exchange" if ex is not None else "") +
                    "), star_decode_advance once per token, 32 layers in one CUDA graph per token"),
           "launches_per_token": n_layers + 1 if finish is not None else 2 * n_layers + 1}
    del pool, g
    torch.cuda.empty_cache()
    return res


def decode_sweep(dev, hq, hkv, d, hbm_peak, n_tokens=64, cap_gib=64.0):
    """BASELINE configs[4]: batch B in {1..32} x 64 generated tokens over S in {32K..1M}
    cached tokens, split-KV + LSE merge at G in {1, 2, 4, 8} ranks, one layer.

    A rank holds S/G cached rows per sequence, so the per-rank work of (B, S, G) is the
    (B, S/G) point: per token, star_kv_append of the B new rows (the query rank's append,
    device counters) + K2 over the B sequences' paged caches, captured in one CUDA graph and
    replayed for the 64 generated tokens (the caches grow by one row per token).  For G > 1
    the cross-rank combine is the merge of G (out, lse) partials, timed here as K3 over G
    parts (its NVLink transport is the peer exchange).  Points whose per-rank
    cache exceeds cap_gib are skipped (B = 32 x 1M at G = 1 is 128 GiB)."""
    import torch

    from paper_2411_17116_b200 import ops

    page = 128
    LPT = 8  # fused decode launches per graph step (layers sharing one star_decode_advance)
    Bs, Ss, Gs = (1, 2, 4, 8, 16, 32), (32768, 131072, 262144, 1048576), (1, 2, 4, 8)
    kern = {}
    for B in Bs:
        for rows in sorted({S // G for S in Ss for G in Gs}):
            gib = B * rows * hkv * d * 2 * 2 / 2 ** 30
            if gib > cap_gib:
                continue
            pps = -(-(rows + n_tokens) // page)
            # L2-cold: a cache smaller than 512 MiB is replicated (one copy per launch, cycled)
            # so every launch streams its K/V from HBM, as distinct layers do
            cache_b = B * pps * page * hkv * d * 2 * 2
            n_c = 1 if cache_b >= 512 * 2 ** 20 else -(-512 * 2 ** 20 // cache_b)
            lpt = max(LPT, n_c)
            caches = []
            for ci in range(n_c):
                kp = torch.empty((B * pps, hkv, page, d), dtype=torch.bfloat16, device=dev)
                vp = torch.empty_like(kp)
                ops.prng_fill(None, 21 + 2 * ci, out=kp.view(-1))
                ops.prng_fill(None, 22 + 2 * ci, out=vp.view(-1))
                caches.append((kp, vp))
            table = torch.arange(B * pps, dtype=torch.int32, device=dev).view(B, pps)
            q = ops.prng_fill((B, 1, hq, d), 23, 1, 1.0, torch.bfloat16, dev)
            kn = ops.prng_fill((B, hkv, d), 24, 1, 1.0, torch.bfloat16, dev)
            vn = ops.prng_fill((B, hkv, d), 25, 1, 1.0, torch.bfloat16, dev)
            pos = torch.full((B,), rows, dtype=torch.int64, device=dev)
            kv_len = torch.full((B,), rows, dtype=torch.int32, device=dev)
            ws = ops.Phase2Workspace()
            maxk = rows + n_tokens
            rtab = ops.DecodeRope(rows, n_tokens + 8, d, 10000.0, B, dev)
            rtab.prime(pos)

            def step():
                # LPT layers' worth of fused decode launches over this cache (each attends
                # over kv_len + 1 rows and writes the token's row), then the once-per-token
                # counter / position advance — per layer = step / LPT, as in a model step
                for li in range(lpt):
                    kp, vp = caches[li % n_c]
                    ops.phase2_decode(q.view(B, hq, d), kn, vn, pos, kp, vp, table, kv_len, maxk,
                                      table=rtab, workspace=ws)
                ops.decode_advance(kv_len, pos, rope=rtab)

            step()
            side = torch.cuda.Stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
                step()
            torch.cuda.current_stream(dev).wait_stream(side)
            kv_len.fill_(rows)
            pos.fill_(rows)
            rtab.prime(pos)
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(n_tokens):
                g.replay()
            e1.record()
            torch.cuda.synchronize(dev)
            us = e0.elapsed_time(e1) / n_tokens / lpt * 1e3
            nbytes = B * (rows + n_tokens / 2) * hkv * d * 2 * 2  # mean cache over the 64 tokens
            kern[(B, rows)] = (us, nbytes / us / 1e3)
            del caches, g
            torch.cuda.empty_cache()
    merge_us = {}
    for B in Bs:
        for G in Gs[1:]:
            outs = ops.prng_fill((G, B * hq, d), 26, 1, 1.0, torch.float32, dev)
            lses = ops.prng_fill((G, B * hq), 27, 1, 1.0, torch.float32, dev)
            ops.merge(outs, lses)
            torch.cuda.synchronize(dev)
            side = torch.cuda.Stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            gm = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side), torch.cuda.graph(gm, stream=side):
                for _ in range(20):
                    ops.merge(outs, lses)
            torch.cuda.current_stream(dev).wait_stream(side)
            gm.replay()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                gm.replay()
            e1.record()
            torch.cuda.synchronize(dev)
            merge_us[(B, G)] = e0.elapsed_time(e1) / 100 * 1e3
            del gm
    out = []
    for B in Bs:
        for S in Ss:
            for G in Gs:
                k = kern.get((B, S // G))
                if k is None:
                    out.append({"batch": B, "cached_tokens": S, "ranks": G,
                                "skipped": f"per-rank cache > {cap_gib:.0f} GiB"})
                    continue
                out.append({"batch": B, "cached_tokens": S, "ranks": G, "rows_per_rank": S // G,
                            "us_per_token_per_layer": k[0], "gbs": k[1],
                            "frac_of_measured_hbm": k[1] / hbm_peak,
                            "merge_us": merge_us.get((B, G))})
    return {"points": out, "tokens": n_tokens,
            "timing": "per (B, S/G): CUDA graph of max(8, copies) star_phase2_decode launches (RoPE + append "
                      "of the B new rows inside K2 over the B paged caches, one per layer) + one "
                      "star_decode_advance, replayed for 64 generated tokens; value per layer = "
                      "graph / launches; every launch reads its K/V from HBM (caches under 512 MiB are "
                      "replicated and cycled, L2-cold); merge_us = K3 over G partials "
                      "(graph-replayed launches)"}


def cfg1_session(dev):
    """BASELINE configs[0] end to end through the drop-in API (start_session + 16 greedy
    decode steps, the reference's tiny model at 4 hosts, fp32 check mode as the reference):
    wall time per phase and whether the tokens equal the committed reference golden
    (tests/golden/model_tiny_s0.npz, produced by running the reference)."""
    import torch

    import paper_2411_17116_b200 as S

    g = np.load(os.path.join(ROOT, "tests", "golden", "model_tiny_s0.npz"))
    doc = json.loads(str(g["doc"]))
    md = doc["model"]
    prev = S.default_dtype()
    S.set_default_dtype("float32")
    tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        w = S.init_model(S.ModelConfig(d_model=md["d_model"], heads=md["heads"],
                                       layers=md["layers"], seed=md["seed"]))
        plan = S.partition(doc["sequence_len"], doc["block_size"], doc["hosts"])
        spec = S.AnchorSpec(anchor_len=doc["anchor"]["anchor_len"])
        toks = list(g["context_tokens"]) + list(g["query_tokens"])
        salt = 0xA17C4B10C4ED5EED
        res = None
        for _ in range(2):  # the first pass warms the library and the allocator
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            logits, sess = S.start_session(w, toks, plan, spec, prng=S.Prng(doc["seed"] ^ salt))
            torch.cuda.synchronize(dev)
            t1 = time.perf_counter()
            gen = S.decode(sess, doc["n_generate"])
            torch.cuda.synchronize(dev)
            t2 = time.perf_counter()
            S.decode(sess, 48)  # same session, graph already captured: steady state
            torch.cuda.synchronize(dev)
            t3 = time.perf_counter()
            res = {"workload": "configs[0]: tiny model (2 layers, 4 heads, d 64), 4K context, "
                               "block = anchor 1K, 4 simulated hosts, 32-token query + 16 greedy "
                               "tokens, fp32 check mode",
                   "start_session_ms": (t1 - t0) * 1e3,
                   "decode_ms_per_token": (t2 - t1) * 1e3 / doc["n_generate"],
                   "decode_note": "decode() of the 16 reference tokens, including the first "
                                  "(eager) step and the one-time CUDA-graph capture",
                   "decode_steady_ms_per_token": (t3 - t2) * 1e3 / 48,
                   "tokens_equal_reference": [int(t) for t in gen] == [int(t) for t in g["generated"]],
                   "reference_cpu_note": "SURVEY §8d: the reference's start_session ≈2.2 s and "
                                         "≈6.4 ms per decoded token on 8 CPU cores"}
        return res
    finally:
        S.set_default_dtype(prev)
        torch.backends.cuda.matmul.allow_tf32 = tf32


def config_shares(dev, tensor_peak):
    """BASELINE configs[1..3] phase 1 on the busiest GPU of an 8-GPU run: its share is one
    anchor-augmented block (b own rows + a anchor rows), so K1 is timed on one such segment
    at each config's heads.  FLOPs = m(m+1)/2 pairs x Hq x 4d."""
    import torch

    from paper_2411_17116_b200 import ops

    out = []
    for name, b, a, hq, hkv, L in (("cfg2 Llama-3.1-8B 128K, b=a=16K", 16384, 16384, 32, 8, 131072),
                                   ("cfg3 Llama-3.1-8B 1M, b=a=128K", 131072, 131072, 32, 8, 1 << 20),
                                   ("cfg4 Llama-3.1-70B 256K, b=a=32K", 32768, 32768, 64, 8, 262144)):
        d = 128
        m = a + b
        q = ops.prng_fill((m, hq, d), 31, 1, 1.0, torch.bfloat16, dev)
        k = ops.prng_fill((m, hkv, d), 32, 1, 1.0, torch.bfloat16, dev)
        v = ops.prng_fill((m, hkv, d), 33, 1, 1.0, torch.bfloat16, dev)
        o = torch.empty_like(q)
        ops.phase1_fwd(q, k, v, [0, m], out=o)
        torch.cuda.synchronize(dev)
        reps = 2 if m > 100000 else 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            ops.phase1_fwd(q, k, v, [0, m], out=o)
        e1.record()
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / reps
        flops = m * (m + 1) // 2 * hq * 4 * d
        tf = flops / (ms * 1e-3) / 1e12
        out.append({"config": name, "gpu_share": f"one {m}-row augmented block x {hq} q heads "
                    f"(the last block: busiest GPU at G = 8)", "k1_ms": ms,
                    "flops": flops, "tflops": tf, "frac_of_measured_sustained": tf / tensor_peak,
                    "context_tokens_per_s_at_8gpu_bound": L / (ms * 1e-3)})
        del q, k, v, o
        torch.cuda.empty_cache()
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-sweep", action="store_true")
    args = p.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus < 1:
        p.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch this command under torch.distributed.run
        import socket

        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
