# experiment batch G: K2 cluster (DSMEM) split merge
mkdir -p gpurun_out
O=gpurun_out/exp_g.log
{
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_fullsize_gpu.py tests/test_model_gpu.py tests/test_dist_gpu.py -x -q -k "phase2 or merge or decode or session or dist" 2>&1 | tail -3
for nc in 0 1; do
  if [ $nc = 1 ]; then export STAR_K2_NO_CLUSTER=1; fi
  echo "NO_CLUSTER=$nc"
  for rows in 16384 32768 131072 1048576; do timeout 120 python tools/decode_bench.py --rows $rows --splits 0 12 16 --iters 200; done
  timeout 120 python tools/decode_bench.py --rows 32768 --batch 2 --splits 0 --iters 100
  timeout 120 python tools/decode_bench.py --rows 32768 --batch 4 --splits 0 --iters 100
done
unset STAR_K2_NO_CLUSTER
timeout 300 python tools/k2_err.py
} > $O 2>&1
