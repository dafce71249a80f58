mkdir -p gpurun_out
O=gpurun_out/qe.log
{
export STAR_EXCHANGE_TIMEOUT_S=20
timeout -s KILL 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "phase2" 2>&1 | tail -15
timeout 300 python tools/query_bench.py
echo "QE off"; STAR_K2_QE=0 timeout 300 python tools/query_bench.py
} > $O 2>&1
