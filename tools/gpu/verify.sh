# quick verification: full GPU test suite + smoke + decode sweep
mkdir -p gpurun_out
TAG=${1:-verify}
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/${TAG}_pytest.log 2>&1
for rows in 16384 131072; do timeout 120 python tools/decode_bench.py --rows $rows --splits 0 --iters 200; done >> gpurun_out/${TAG}_pytest.log 2>&1
