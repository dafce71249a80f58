mkdir -p gpurun_out
make -C paper_2411_17116_b200/csrc trace -j8 > /dev/null 2>&1
for v in 9 20 13; do
  echo "== SM=$v" >> gpurun_out/r02p_k1_trace.log
  STAR_K1_SM=$v timeout 60 python tools/k1_trace.py 2>&1 | tail -1 >> gpurun_out/r02p_k1_trace.log
done
