# experiment batch E: split P hand-off (variant 3) parity + speed + trace
mkdir -p gpurun_out
O=gpurun_out/exp_e.log
{
STAR_K1_VARIANT=3 timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_fullsize_gpu.py -x -q -k "phase1" 2>&1 | tail -3
for cfg in "STAR_K1_VARIANT=1" "STAR_K1_VARIANT=3" "STAR_K1_VARIANT=3 STAR_K1_SPIN=1" "STAR_K1_VARIANT=1" "STAR_K1_VARIANT=3"; do
  env $cfg timeout 300 python tools/phase1_bench.py --iters 5
done
for cfg in "STAR_K1_VARIANT=3"; do env $cfg timeout 300 python tools/k1_trace.py; done
} > $O 2>&1
