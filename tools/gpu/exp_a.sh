# experiment batch A: K2 short-context sweep, SFU microbench, K1 knob A/B + trace
mkdir -p gpurun_out
O=gpurun_out/exp_a.log
{
./tools/ubench/mufu
for rows in 16384 32768 131072; do
  timeout 120 python tools/decode_bench.py --rows $rows --splits 0 9 16 18 36 --iters 200
  STAR_K2_EXPERIMENT_NOFIX=1 timeout 120 python tools/decode_bench.py --rows $rows --splits 18 --iters 200
done
for cfg in "STAR_K1_ONEP=1" "STAR_K1_ONEP=1 STAR_K1_POLY=1" "STAR_K1_ONEP=1 STAR_K1_SEQ=0" "STAR_K1_ONEP=0"; do
  env $cfg timeout 300 python tools/phase1_bench.py --iters 5
done
for cfg in "STAR_K1_ONEP=1" "STAR_K1_ONEP=1 STAR_K1_POLY=1"; do env $cfg timeout 300 python tools/k1_trace.py; done
} > $O 2>&1
