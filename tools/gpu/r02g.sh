# K1 softmax variants (STAR_K1_SM): cfg2 layer + trace
mkdir -p gpurun_out
make -C paper_2411_17116_b200/csrc trace -j8 > /dev/null 2>&1
for v in 0 1 2 3 4 5 6 0; do
  STAR_K1_SM=$v timeout 120 python tools/phase1_bench.py --iters 5 >> gpurun_out/r02g_k1_variants.log 2>&1
done
for v in 0 1 2 4; do
  echo "== SM=$v" >> gpurun_out/r02g_k1_trace.log
  STAR_K1_SM=$v timeout 120 python tools/k1_trace.py 2>&1 | tail -1 >> gpurun_out/r02g_k1_trace.log
done
