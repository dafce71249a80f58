set -x
export STAR_EXCHANGE_TIMEOUT_S=5
O=gpurun_out/k2ov
mkdir -p $O
for v in "" "STAR_K2_COOP=0" "STAR_K2_PDL=0" "STAR_K2_COOP=0 STAR_K2_PDL=0" "STAR_K2_FIXUP=atomic"; do
  echo "== $v" >> $O/log
  env $v timeout 120 python tools/k2_overhead.py 256 1024 4096 16384 32768 >> $O/log 2>&1
done
for r in 1024 4096 16384; do
  timeout 60 python tools/k2_trace.py --rows $r >> $O/trace.log 2>&1
  timeout 60 python tools/k2_trace.py --rows $r --decode >> $O/trace.log 2>&1
done
