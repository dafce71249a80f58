mkdir -p gpurun_out
(nproc; free -g; nvidia-smi -L) > gpurun_out/r02zc_host.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r02zc_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02zc_pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02zc_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r02zc_smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/r02zc_bench_n1.json 2> gpurun_out/r02zc_bench_n1.err
timeout -s KILL 600 python tools/yardstick.py > gpurun_out/r02zc_yardstick.json 2> gpurun_out/r02zc_yardstick.err
