mkdir -p gpurun_out
O=gpurun_out/fused.log
{
export STAR_EXCHANGE_TIMEOUT_S=20
timeout -s KILL 900 python -m pytest tests/test_exchange_gpu.py tests/test_dist_gpu.py tests/test_kernels_gpu.py -x -q 2>&1 | tail -5
timeout 200 python tools/exchange_bench.py
timeout 100 python tools/k2_trace.py --rows 16384
timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --no-sweep 2>&1 | tail -1 | cut -c1-100
} > $O 2>&1
