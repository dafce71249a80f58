mkdir -p gpurun_out
make -C paper_2411_17116_b200/csrc trace -j8 > /dev/null 2>&1
for r in 4096 16384; do
  timeout 60 python tools/k2_trace.py --rows $r >> gpurun_out/r02zb_k2_trace.log 2>&1
  timeout 60 python tools/k2_trace.py --rows $r --decode >> gpurun_out/r02zb_k2_trace.log 2>&1
done
