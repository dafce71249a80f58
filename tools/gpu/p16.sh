mkdir -p gpurun_out
O=gpurun_out/p16.log
{
STAR_K2_QE=0 python tools/qe_debug.py x 32 3000,1500
STAR_K2_QE=1 STAR_K2Q_P16=1 python tools/qe_debug.py --cmp 32 3000,1500 | tail -4
STAR_K2Q_P16=1 timeout -s KILL 600 python -m pytest tests/test_kernels_gpu.py -x -q -k phase2 2>&1 | tail -2
STAR_K2Q_P16=1 QB_ROWS=16384,131072 QB_LQ=8,32 timeout 300 python tools/query_bench.py
QB_ROWS=16384,131072 QB_LQ=8,32 timeout 300 python tools/query_bench.py
} > $O 2>&1
