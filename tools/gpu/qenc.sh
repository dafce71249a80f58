mkdir -p gpurun_out
O=gpurun_out/qenc.log
{
timeout -s KILL 900 python -m pytest tests/test_kernels_gpu.py tests/test_exchange_gpu.py tests/test_model_gpu.py tests/test_dist_gpu.py -x -q 2>&1 | tail -3
timeout 300 python tools/query_bench.py
} > $O 2>&1
echo OLD >> $O; STAR_LIB_PATH=$PWD/tools/oldlib/libstar_attn.so timeout 300 python tools/query_bench.py >> $O 2>&1
