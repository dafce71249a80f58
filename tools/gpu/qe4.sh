mkdir -p gpurun_out
O=gpurun_out/qe4.log
{
timeout 300 python tools/k2q_trace.py | tail -1
QB_ROWS=16384,131072 QB_LQ=8,32 timeout 300 python tools/query_bench.py
timeout -s KILL 600 python -m pytest tests/test_kernels_gpu.py tests/test_exchange_gpu.py -x -q -k "phase2 or exchange" 2>&1 | tail -2
} > $O 2>&1
