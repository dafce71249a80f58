mkdir -p gpurun_out
timeout -s KILL 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r02d_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02d_pytest_gpu.log
timeout -s KILL 900 python bench.py > gpurun_out/r02d_bench_n1.json 2> gpurun_out/r02d_bench_n1.err
timeout -s KILL 600 python tools/yardstick.py > gpurun_out/r02d_yardstick.json 2> gpurun_out/r02d_yardstick.err
