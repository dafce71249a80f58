mkdir -p gpurun_out
O=gpurun_out/qe.log
{
export STAR_EXCHANGE_TIMEOUT_S=20
STAR_K2_QE=0 python tools/qe_debug.py; STAR_K2_QE=1 python tools/qe_debug.py --cmp | tail -3
timeout -s KILL 900 python -m pytest tests/test_kernels_gpu.py tests/test_exchange_gpu.py tests/test_fullsize_gpu.py tests/test_model_gpu.py -x -q 2>&1 | tail -4
timeout 300 python tools/query_bench.py
} > $O 2>&1
