mkdir -p gpurun_out
for v in 0 4 5 0 4 5; do
  STAR_K1_SM=$v timeout 60 python tools/phase1_bench.py --iters 5 >> gpurun_out/r02u_k1_variants.log 2>&1
done
STAR_K1_SEQ=0 timeout 60 python tools/phase1_bench.py --iters 5 >> gpurun_out/r02u_k1_variants.log 2>&1
STAR_K1_SEQ=0 timeout 60 python tools/phase1_bench.py --iters 5 >> gpurun_out/r02u_k1_variants.log 2>&1
for v in 4 5; do STAR_K1_SM=$v timeout 90 python tools/k1_accuracy.py >> gpurun_out/r02u_k1_accuracy.log 2>&1; done
