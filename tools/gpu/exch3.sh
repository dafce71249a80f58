mkdir -p gpurun_out
O=gpurun_out/exch3.log
{
export STAR_EXCHANGE_TIMEOUT_S=20
timeout -s KILL 600 python -m pytest tests/test_exchange_gpu.py tests/test_dist_gpu.py -x -q 2>&1 | tail -5
timeout -s KILL 200 python tools/exchange_bench.py
STAR_EXCHANGE_PDL=0 timeout -s KILL 200 python tools/exchange_bench.py
} > $O 2>&1
