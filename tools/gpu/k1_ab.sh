# K1 knob A/B at cfg2 (+ the phase-1 kernel tests) — run under gpurun
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "phase1" 2>&1 | tail -2
for cfg in ${K1_CFGS:-"STAR_K1_ONEP=0" "STAR_K1_ONEP=1" "STAR_K1_ONEP=1 STAR_K1_SEQ=0" "STAR_K1_ONEP=1 STAR_K1_POLY=1"}; do
  env $cfg timeout 300 python tools/phase1_bench.py --iters 5
done
for cfg in ${K1_TRACE:-"STAR_K1_ONEP=1"}; do env $cfg timeout 300 python tools/k1_trace.py | tail -1; done
