mkdir -p gpurun_out
(nproc; free -g; nvidia-smi -L) > gpurun_out/r02e_host.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r02e_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02e_pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02e_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r02e_smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/r02e_bench_n1.json 2> gpurun_out/r02e_bench_n1.err
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02e_bench_ref_n1.json 2> gpurun_out/r02e_bench_ref_n1.err
timeout -s KILL 600 python tools/yardstick.py > gpurun_out/r02e_yardstick.json 2> gpurun_out/r02e_yardstick.err
