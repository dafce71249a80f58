mkdir -p gpurun_out
(nproc; free -g; lscpu | head -20) > gpurun_out/r02b_host.txt 2>&1
timeout -s KILL 1800 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r02b_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02b_pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.log 2>&1
timeout -s KILL 900 python bench.py > gpurun_out/r02b_bench_n1.json 2> gpurun_out/r02b_bench_n1.err
