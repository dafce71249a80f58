mkdir -p gpurun_out
O=gpurun_out/k1warp.log
{
for r in 1 2; do timeout 300 python tools/phase1_bench.py --iters 5; done
timeout 300 python tools/k1_trace.py | tail -1
timeout -s KILL 900 python -m pytest tests/test_kernels_gpu.py tests/test_fullsize_gpu.py -x -q -k "phase1 or umma" 2>&1 | tail -2
} > $O 2>&1
