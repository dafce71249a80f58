mkdir -p gpurun_out
O=gpurun_out/exp_k.log
{
timeout 600 python -m pytest tests/test_pipeline_gpu.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --no-cpu-baseline --no-sweep
} > $O 2>&1
