mkdir -p gpurun_out
O=gpurun_out/variants.log
{
export STAR_EXCHANGE_TIMEOUT_S=20
echo "== STAR_K2_QE=0"; STAR_K2_QE=0 timeout -s KILL 600 python -m pytest tests/test_kernels_gpu.py tests/test_exchange_gpu.py -x -q -k "phase2 or exchange" 2>&1 | tail -2
echo "== STAR_K2_FIXUP=atomic"; STAR_K2_FIXUP=atomic timeout -s KILL 600 python -m pytest tests/test_kernels_gpu.py tests/test_exchange_gpu.py tests/test_fullsize_gpu.py -x -q -k "phase2 or exchange or decode" 2>&1 | tail -2
echo "== STAR_EXCHANGE_PDL=0"; STAR_EXCHANGE_PDL=0 timeout -s KILL 600 python -m pytest tests/test_exchange_gpu.py -x -q 2>&1 | tail -2
} > $O 2>&1
