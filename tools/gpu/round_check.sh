# Full round check on one B200 (run under gpurun): GPU tests, smoke, bench (ours + reference
# arm), the K1 yardstick, and the ncu launch list + full captures.  Usage: round_check.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
(nproc; free -g; nvidia-smi -L) > gpurun_out/${TAG}_host.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/${TAG}_bench_n1.json 2> gpurun_out/${TAG}_bench_n1.err
timeout -s KILL 900 python bench.py --impl reference --steps 2 > gpurun_out/${TAG}_bench_ref_n1.json 2> gpurun_out/${TAG}_bench_ref_n1.err
timeout -s KILL 600 python tools/yardstick.py > gpurun_out/${TAG}_yardstick.json 2> gpurun_out/${TAG}_yardstick.err
bash tools_profile.sh ${TAG}
