mkdir -p gpurun_out
for v in 20 21 22 23 20 21 22 23; do
  STAR_K1_SM=$v timeout 60 python tools/phase1_bench.py --iters 5 >> gpurun_out/r02s_k1_variants.log 2>&1
done
for q in 1 2; do
  rm -rf paper_2411_17116_b200/csrc/build_trace paper_2411_17116_b200/libstar_attn_trace.so
  make -C paper_2411_17116_b200/csrc trace -j8 TRACE_FLAGS=-DSTAR_K1_TRQ=$q > /dev/null 2>&1
  for v in 21; do
    echo "== SM=$v TRQ=$q" >> gpurun_out/r02s_k1_trace.log
    STAR_K1_SM=$v timeout 60 python tools/k1_trace.py 2>&1 | tail -1 >> gpurun_out/r02s_k1_trace.log
  done
done
STAR_K1_SM=21 timeout 90 python tools/k1_accuracy.py >> gpurun_out/r02s_k1_accuracy.log 2>&1
