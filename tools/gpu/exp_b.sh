# experiment batch B: K2 fix-up rewrite sweep + parity; K1 variant x spin A/B + traces
mkdir -p gpurun_out
O=gpurun_out/exp_b.log
{
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_fullsize_gpu.py -x -q 2>&1 | tail -3
for rows in 16384 32768 131072; do
  timeout 120 python tools/decode_bench.py --rows $rows --splits 0 16 18 --iters 200
done
for v in 1 3; do for sp in 0 1 2 3; do
  STAR_K1_VARIANT=$v STAR_K1_SPIN=$sp timeout 300 python tools/phase1_bench.py --iters 5
done; done
for cfg in "STAR_K1_VARIANT=3" "STAR_K1_VARIANT=1 STAR_K1_SPIN=1" "STAR_K1_VARIANT=3 STAR_K1_SPIN=1"; do env $cfg timeout 300 python tools/k1_trace.py | tail -1; done
} > $O 2>&1
