mkdir -p gpurun_out
make -C paper_2411_17116_b200/csrc trace -j8 > /dev/null 2>&1
for v in 9 16 17 20 9 16 17 20; do
  STAR_K1_SM=$v timeout 60 python tools/phase1_bench.py --iters 5 >> gpurun_out/r02q_k1_variants.log 2>&1
done
for v in 16 17; do
  echo "== SM=$v" >> gpurun_out/r02q_k1_trace.log
  STAR_K1_SM=$v timeout 60 python tools/k1_trace.py 2>&1 | tail -1 >> gpurun_out/r02q_k1_trace.log
  STAR_K1_SM=$v timeout 90 python tools/k1_accuracy.py >> gpurun_out/r02q_k1_accuracy.log 2>&1
done
