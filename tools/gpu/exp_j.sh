# K1 v3 (P in smem, early S): parity, speed, trace
mkdir -p gpurun_out
O=gpurun_out/exp_j.log
{
STAR_K1_V3=1 timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_fullsize_gpu.py -x -q -k "phase1" 2>&1 | tail -3
for cfg in "STAR_K1_V3=0" "STAR_K1_V3=1" "STAR_K1_V3=1 STAR_K1_SEQ=0" "STAR_K1_V3=0" "STAR_K1_V3=1"; do
  env $cfg timeout 300 python tools/phase1_bench.py --iters 5
done
for cfg in "STAR_K1_V3=1" "STAR_K1_V3=1 STAR_K1_SEQ=0"; do env $cfg timeout 300 python tools/k1_trace.py; done
./tools/ubench/mufu | grep -i "f16\|bf16x2"
} > $O 2>&1
