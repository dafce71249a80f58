mkdir -p gpurun_out
O=gpurun_out/k1knobs.log
{
for cfg in "STAR_K1_SEQ=1" "STAR_K1_SEQ=0" "STAR_K1_SPEC=1" "STAR_K1_SEQ=1" "STAR_K1_POLY=1"; do
  env $cfg timeout 300 python tools/phase1_bench.py --iters 5
done
} > $O 2>&1
