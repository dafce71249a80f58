# K1: 12-warp setmaxnreg layout variants (STAR_K1_SM 7-10) vs 10-warp (0, 4)
mkdir -p gpurun_out
make -C paper_2411_17116_b200/csrc trace -j8 > /dev/null 2>&1
for v in 0 4 7 8 9 10 4 0; do
  STAR_K1_SM=$v timeout 120 python tools/phase1_bench.py --iters 5 >> gpurun_out/r02j_k1_variants.log 2>&1
done
for v in 4 8 9 10; do
  echo "== SM=$v" >> gpurun_out/r02j_k1_trace.log
  STAR_K1_SM=$v timeout 120 python tools/k1_trace.py 2>&1 | tail -1 >> gpurun_out/r02j_k1_trace.log
  STAR_K1_SM=$v timeout 300 python tools/k1_accuracy.py >> gpurun_out/r02j_k1_accuracy.log 2>&1
done
