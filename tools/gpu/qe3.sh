mkdir -p gpurun_out
O=gpurun_out/qe3.log
{
export STAR_EXCHANGE_TIMEOUT_S=20
timeout -s KILL 600 python -m pytest tests/test_kernels_gpu.py tests/test_exchange_gpu.py -x -q -k "phase2 or exchange" 2>&1 | tail -3
QB_ROWS=16384,131072 QB_LQ=8,16,32 timeout 300 python tools/query_bench.py
} > $O 2>&1
