# peer exchange bring-up: exchange + dist + phase-2 kernel tests, bench N=1, 2-rank gloo bench on one GPU
mkdir -p gpurun_out
O=gpurun_out/exch.log
{
export STAR_EXCHANGE_TIMEOUT_S=20
timeout -s KILL 600 python -m pytest tests/test_exchange_gpu.py tests/test_kernels_gpu.py -x -q -k "exchange or phase2 or merge" 2>&1 | tail -30
timeout -s KILL 600 python -m pytest tests/test_dist_gpu.py -x -q 2>&1 | tail -30
timeout -s KILL 600 python bench.py --no-e2e --no-cpu-baseline --no-sweep 2>&1 | tail -3
STAR_BENCH_BACKEND=gloo timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep 2>&1 | tail -5
} > $O 2>&1
