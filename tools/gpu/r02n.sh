mkdir -p gpurun_out
make -C paper_2411_17116_b200/csrc trace -j8 > /dev/null 2>&1
STAR_K1_SM=17 timeout 60 python tools/phase1_bench.py --L 4096 --b 2048 --iters 1 > gpurun_out/r02n_dbg.log 2>&1; echo "rc=$?" >> gpurun_out/r02n_dbg.log
for v in 9 13 14 15 16 13 9; do
  STAR_K1_SM=$v timeout 60 python tools/phase1_bench.py --iters 5 >> gpurun_out/r02n_k1_variants.log 2>&1
done
for v in 13 14 16; do
  echo "== SM=$v" >> gpurun_out/r02n_k1_trace.log
  STAR_K1_SM=$v timeout 60 python tools/k1_trace.py 2>&1 | tail -1 >> gpurun_out/r02n_k1_trace.log
  STAR_K1_SM=$v timeout 90 python tools/k1_accuracy.py >> gpurun_out/r02n_k1_accuracy.log 2>&1
done
