# experiment batch C: K2 PLO knob (speed + error), softmax ubench, K1 spread-poly variants
mkdir -p gpurun_out
O=gpurun_out/exp_c.log
{
./tools/ubench/softmax_row
for plo in 1 0; do
  export STAR_K2_PLO=$plo
  for rows in 16384 131072; do timeout 120 python tools/decode_bench.py --rows $rows --splits 0 16 --iters 200; done
  timeout 300 python tools/k2_err.py
  timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_fullsize_gpu.py -x -q -k phase2 2>&1 | tail -2
done
unset STAR_K2_PLO
for v in 1 4 5 2; do STAR_K1_VARIANT=$v STAR_K1_SPIN=1 timeout 300 python tools/phase1_bench.py --iters 5; done
for v in 4 5; do STAR_K1_VARIANT=$v STAR_K1_SPIN=1 timeout 300 python tools/k1_trace.py | tail -1; done
STAR_K1_VARIANT=4 timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k phase1 2>&1 | tail -2
} > $O 2>&1
