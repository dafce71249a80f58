# K1 split hand-off / sum / poly variants: cfg2 timing, accuracy vs fp32 kernel, trace
mkdir -p gpurun_out
make -C paper_2411_17116_b200/csrc trace -j8 > /dev/null 2>&1
for v in 0 1 2 3 4 5 6 0; do
  STAR_K1_SM=$v timeout 120 python tools/phase1_bench.py --iters 5 >> gpurun_out/r02h_k1_variants.log 2>&1
done
for v in 0 3 4 5; do
  echo "== SM=$v" >> gpurun_out/r02h_k1_trace.log
  STAR_K1_SM=$v timeout 120 python tools/k1_trace.py 2>&1 | tail -1 >> gpurun_out/r02h_k1_trace.log
  STAR_K1_SM=$v timeout 300 python tools/k1_accuracy.py >> gpurun_out/r02h_k1_accuracy.log 2>&1
done
