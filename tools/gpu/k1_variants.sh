# K1 form A/B (STAR_K1_SM values, clock-normalised by tools/phase1_bench.py) + clock64 traces
# of two lane quarters.  Usage: k1_variants.sh TAG "0 1 2 3"
TAG=${1:-r02}; VARS=${2:-"0 1 2 3"}
mkdir -p gpurun_out
for v in $VARS $VARS; do
  STAR_K1_SM=$v timeout 60 python tools/phase1_bench.py --iters 5 >> gpurun_out/${TAG}_k1_variants.log 2>&1
done
for q in 1 2; do
  rm -rf paper_2411_17116_b200/csrc/build_trace paper_2411_17116_b200/libstar_attn_trace.so
  make -C paper_2411_17116_b200/csrc trace -j8 TRACE_FLAGS=-DSTAR_K1_TRQ=$q > /dev/null 2>&1
  for v in $VARS; do
    echo "== SM=$v TRQ=$q" >> gpurun_out/${TAG}_k1_trace.log
    STAR_K1_SM=$v timeout 60 python tools/k1_trace.py 2>&1 | tail -1 >> gpurun_out/${TAG}_k1_trace.log
  done
done
for v in $VARS; do STAR_K1_SM=$v timeout 90 python tools/k1_accuracy.py >> gpurun_out/${TAG}_k1_accuracy.log 2>&1; done
