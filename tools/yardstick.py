"""K1 yardstick: the container's own sm100 attention kernels on K1's workload unit.

One causal self-attention over a 32,768-row augmented block (cfg2's unit: b + a rows),
32 q / 8 kv heads, head_dim 128, bf16, on the same GPU in the same process as K1:
  * ours     — paper_2411_17116_b200.ops.phase1_fwd (tcgen05 K1)
  * cudnn    — torch SDPA, cuDNN backend (enable_gqa)
  * flash    — torch SDPA, flash backend
  * fa2      — flash_attn 2.8 flash_attn_func (GQA native)
  * flashinfer — flashinfer.single_prefill_with_kv_cache, each backend it accepts, and
    flashinfer.prefill.fmha_varlen (its CUTLASS sm100a FMHA, JIT-built on first use)
FLOPs = m(m+1)/2 pairs x Hq x 4d (the causal triangle), timed with CUDA events
over back-to-back launches after warm-up.  Output: one JSON line (informational; library
kernels are the yardstick, not the product).

Usage: python tools/yardstick.py [rows]
"""

import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    from bench import ClockSampler
    from paper_2411_17116_b200 import ops

    m = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    hq, hkv, d = 32, 8, 128
    dev = torch.device("cuda", 0)
    q = ops.prng_fill((m, hq, d), 31, 1, 1.0, torch.bfloat16, dev)
    k = ops.prng_fill((m, hkv, d), 32, 1, 1.0, torch.bfloat16, dev)
    v = ops.prng_fill((m, hkv, d), 33, 1, 1.0, torch.bfloat16, dev)
    flops = m * (m + 1) // 2 * hq * 4 * d
    res = {"rows": m, "heads_q": hq, "heads_kv": hkv, "head_dim": d, "flops": flops, "kernels": {}}
    ref = torch.empty_like(q)
    ops.phase1_fwd(q, k, v, [0, m], out=ref)
    # accuracy yardstick: the fp32 CUDA-core check kernel on the same bf16 inputs
    chk, _ = ops.phase1_fwd_check(q, k, v, [0, m], want_lse=False)

    def accuracy(o):
        """normwise error per (128-row block, head) vs the fp32 check kernel: max, p99.9,
        share of blocks above 2e-3; and the worst per-head Frobenius relative error."""
        o = o.float()
        nb = m // 128
        num = (o[:nb * 128] - chk[:nb * 128]).abs().view(nb, 128, hq, d).amax(dim=(1, 3))
        den = chk[:nb * 128].abs().view(nb, 128, hq, d).amax(dim=(1, 3))
        e = (num / den).flatten()
        fro = ((o - chk).pow(2).sum(dim=(0, 2)).sqrt() / chk.pow(2).sum(dim=(0, 2)).sqrt()).max()
        return {"block_normwise_max": float(e.max()),
                "block_normwise_p999": float(e.quantile(0.999)),
                "share_blocks_over_2e-3": float((e > 2e-3).float().mean()),
                "frobenius_rel_max_head": float(fro)}

    def record(name, fn, check=None):
        t0 = time.time()
        try:
            out = fn()
            torch.cuda.synchronize()
            err = None
            acc = None
            if check is not None:
                o = check(out)
                err = float((o.float() - ref.float()).abs().max() / ref.float().abs().max())
                acc = accuracy(o)
            ms = timed(fn)
            res["kernels"][name] = {"ms": ms, "tflops": flops / (ms * 1e-3) / 1e12,
                                    "normwise_vs_ours": err, "accuracy_vs_fp32": acc,
                                    "setup_s": time.time() - t0}
        except Exception as exc:  # noqa: BLE001 - a yardstick that does not run is reported
            torch.cuda.synchronize()
            res["kernels"][name] = {"error": f"{type(exc).__name__}: {str(exc)[:300]}"}

    with ClockSampler(0) as clk:
        o = torch.empty_like(q)
        record("ours_k1", lambda: ops.phase1_fwd(q, k, v, [0, m], out=o), check=lambda out: o)
        o32 = torch.empty(q.shape, dtype=torch.float32, device=dev)
        record("ours_k1_f32out", lambda: ops.phase1_fwd(q, k, v, [0, m], out=o32),
               check=lambda out: o32)
        qt, kt, vt = (x.transpose(0, 1).unsqueeze(0) for x in (q, k, v))  # [1, H, S, D] views
        from torch.nn.attention import SDPBackend, sdpa_kernel
        import torch.nn.functional as F

        for name, be in (("torch_sdpa_cudnn", SDPBackend.CUDNN_ATTENTION),
                         ("torch_sdpa_flash", SDPBackend.FLASH_ATTENTION),
                         ("torch_sdpa_efficient", SDPBackend.EFFICIENT_ATTENTION)):
            def run(be=be):
                with sdpa_kernel([be]):
                    return F.scaled_dot_product_attention(qt, kt, vt, is_causal=True, enable_gqa=True)
            record(name, run, check=lambda out: out[0].transpose(0, 1))
        try:
            from flash_attn import flash_attn_func

            record("flash_attn2", lambda: flash_attn_func(q.unsqueeze(0), k.unsqueeze(0),
                                                          v.unsqueeze(0), causal=True),
                   check=lambda out: out[0])
        except ImportError as exc:
            res["kernels"]["flash_attn2"] = {"error": str(exc)}
        try:
            import flashinfer

            for be in ("trtllm-gen", "cutlass", "fa3", "fa2"):
                record(f"flashinfer_{be}",
                       lambda be=be: flashinfer.single_prefill_with_kv_cache(q, k, v, causal=True,
                                                                             backend=be),
                       check=lambda out: out)
            from flashinfer.prefill import fmha_varlen

            offs = torch.tensor([0, m], dtype=torch.int32, device=dev)
            first = lambda out: out[0] if isinstance(out, tuple) else out  # noqa: E731
            record("flashinfer_cutlass_sm100_fmha",
                   lambda: fmha_varlen(q, k, v, offs, offs, causal=True),
                   check=first)
        except ImportError as exc:
            res["kernels"]["flashinfer"] = {"error": str(exc)}
    res["clocks"] = clk.summary()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
