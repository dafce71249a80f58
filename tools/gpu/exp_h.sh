mkdir -p gpurun_out
O=gpurun_out/exp_h.log
{
export STAR_K2_VERBOSE=1
timeout 120 python tools/decode_bench.py --rows 16384 --splits 0 8 12 16 --iters 50
timeout 120 python tools/decode_bench.py --rows 131072 --splits 0 8 --iters 50
timeout 120 python tools/decode_bench.py --rows 32768 --batch 4 --splits 0 --iters 50
} > $O 2>&1
