mkdir -p gpurun_out
O=gpurun_out/exp_m.log
{
timeout -s KILL 600 python -m pytest tests/test_kernels_gpu.py tests/test_pipeline_gpu.py -x -q -k "range or pipeline" 2>&1 | tail -3
export STAR_BENCH_BACKEND=gloo STAR_BENCH_HANG_DUMP=200 MASTER_ADDR=127.0.0.1 MASTER_PORT=29533 WORLD_SIZE=2
for r in 0 1; do RANK=$r LOCAL_RANK=0 timeout -s KILL 300 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-sweep --no-e2e > gpurun_out/exp_m_rank$r.log 2>&1 & done
wait
unset STAR_BENCH_BACKEND STAR_BENCH_HANG_DUMP MASTER_ADDR MASTER_PORT WORLD_SIZE
timeout -s KILL 900 python bench.py --no-cpu-baseline --no-sweep
} > $O 2>&1
