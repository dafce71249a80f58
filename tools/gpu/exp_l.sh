mkdir -p gpurun_out
O=gpurun_out/exp_l.log
{
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_fullsize_gpu.py -x -q -k "phase2" 2>&1 | tail -2
for rows in 16384 32768 131072; do timeout 120 python tools/decode_bench.py --rows $rows --splits 0 --iters 400; done
STAR_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-sweep --no-e2e 2>&1 | tail -2
} > $O 2>&1
