mkdir -p gpurun_out
make -C paper_2411_17116_b200/csrc trace -j8 > /dev/null 2>&1
for v in 9 11 18 19 20 9 11 18 19 20; do
  STAR_K1_SM=$v timeout 60 python tools/phase1_bench.py --iters 5 >> gpurun_out/r02o_k1_variants.log 2>&1
done
for v in 9 11 18 19 20; do
  echo "== SM=$v" >> gpurun_out/r02o_k1_trace.log
  STAR_K1_SM=$v timeout 60 python tools/k1_trace.py 2>&1 | tail -1 >> gpurun_out/r02o_k1_trace.log
done
