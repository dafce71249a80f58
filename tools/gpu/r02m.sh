mkdir -p gpurun_out
for v in 9 16 17; do
  echo "== SM=$v" >> gpurun_out/r02m.log
  STAR_K1_SM=$v timeout 60 python tools/phase1_bench.py --L 4096 --b 2048 --iters 1 >> gpurun_out/r02m.log 2>&1
  echo "rc=$?" >> gpurun_out/r02m.log
done
