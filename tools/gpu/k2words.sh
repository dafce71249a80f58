# K2 word-mode split fix-up vs the arrival-counter fix-up; correctness + timing
mkdir -p gpurun_out
O=gpurun_out/k2words.log
{
timeout -s KILL 600 python -m pytest tests/test_kernels_gpu.py tests/test_exchange_gpu.py tests/test_fullsize_gpu.py -x -q -k "phase2 or exchange or decode or merge" 2>&1 | tail -4
for rows in 16384 32768 131072 1048576; do
  echo "rows=$rows words"; timeout 120 python tools/decode_bench.py --rows $rows --splits 0 --iters 200
  echo "rows=$rows atomic"; STAR_K2_FIXUP=atomic timeout 120 python tools/decode_bench.py --rows $rows --splits 0 --iters 200
done
echo "batch 8 x 128K words"; timeout 120 python tools/decode_bench.py --rows 131072 --batch 8 --iters 50
echo "batch 8 x 128K atomic"; STAR_K2_FIXUP=atomic timeout 120 python tools/decode_bench.py --rows 131072 --batch 8 --iters 50
timeout 200 python tools/exchange_bench.py
} > $O 2>&1
timeout 120 python tools/k2_trace.py --rows 16384 >> $O 2>&1
timeout 120 python tools/k2_trace.py --rows 131072 >> $O 2>&1
