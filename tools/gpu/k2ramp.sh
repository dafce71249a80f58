mkdir -p gpurun_out
O=gpurun_out/k2ramp.log
{
timeout -s KILL 600 python -m pytest tests/test_kernels_gpu.py tests/test_exchange_gpu.py tests/test_fullsize_gpu.py -x -q -k "phase2 or exchange or decode" 2>&1 | tail -2
for rows in 16384 32768 131072; do timeout 120 python tools/decode_bench.py --rows $rows --splits 0 --iters 200; done
timeout 100 python tools/k2_trace.py --rows 16384
timeout 200 python tools/exchange_bench.py
} > $O 2>&1
