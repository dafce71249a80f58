mkdir -p gpurun_out
O=gpurun_out/exp_n.log
{
export STAR_BENCH_BACKEND=gloo STAR_BENCH_HANG_DUMP=240 MASTER_ADDR=127.0.0.1 MASTER_PORT=29534 WORLD_SIZE=2
for r in 0 1; do RANK=$r LOCAL_RANK=0 timeout -s KILL 300 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/exp_n_rank$r.log 2>&1 & done
wait
export WORLD_SIZE=4 MASTER_PORT=29535
for r in 0 1 2 3; do RANK=$r LOCAL_RANK=0 timeout -s KILL 300 python bench.py --gpus 4 --steps 3 --warmup 3 --no-cpu-baseline --no-sweep --no-e2e > gpurun_out/exp_n4_rank$r.log 2>&1 & done
wait
} > $O 2>&1
