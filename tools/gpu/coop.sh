mkdir -p gpurun_out
O=gpurun_out/coop.log
{
export STAR_EXCHANGE_TIMEOUT_S=30
timeout -s KILL 900 python -m pytest tests/test_kernels_gpu.py tests/test_exchange_gpu.py tests/test_dist_gpu.py tests/test_fullsize_gpu.py -x -q 2>&1 | tail -3
for rows in 16384 131072; do timeout 120 python tools/decode_bench.py --rows $rows --splits 0 --iters 200; done
timeout 200 python tools/exchange_bench.py
} > $O 2>&1
