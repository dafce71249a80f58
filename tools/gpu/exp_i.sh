mkdir -p gpurun_out
O=gpurun_out/exp_i.log
{
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_fullsize_gpu.py tests/test_model_gpu.py tests/test_dist_gpu.py -x -q -k "phase2 or merge or decode or session or dist" 2>&1 | tail -3
for rows in 16384 32768 131072 1048576; do timeout 120 python tools/decode_bench.py --rows $rows --splits 0 --iters 200; done
STAR_K2_EXPERIMENT_NOFIX=1 timeout 120 python tools/decode_bench.py --rows 16384 --splits 0 --iters 200
timeout 300 python tools/k2_err.py | tail -4
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e
} > $O 2>&1
