mkdir -p gpurun_out
for q in 1 2; do
  rm -rf paper_2411_17116_b200/csrc/build_trace paper_2411_17116_b200/libstar_attn_trace.so
  make -C paper_2411_17116_b200/csrc trace -j8 TRACE_FLAGS=-DSTAR_K1_TRQ=$q > /dev/null 2>&1
  for v in 9 16; do
    echo "== SM=$v TRQ=$q" >> gpurun_out/r02r_k1_trace.log
    STAR_K1_SM=$v timeout 60 python tools/k1_trace.py 2>&1 | tail -1 >> gpurun_out/r02r_k1_trace.log
  done
done
