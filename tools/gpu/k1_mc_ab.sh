# K1 K/V multicast across the head pairs of a q tile (2-CTA cluster) vs the single-CTA form:
# parity tests, then alternating cfg2 timings and a bit-exact output comparison.  Usage: TAG
T=${1:-r02r}
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_kernels_gpu.py tests/test_fuzz_gpu.py tests/test_fullsize_gpu.py -m gpu -q -x -k "phase1 or every_row" > gpurun_out/${T}_k1_mc_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_k1_mc_tests.log
for i in 1 2 3; do
  for v in 0 1; do
    STAR_K1_MC=$v timeout 300 python tools/phase1_bench.py --iters 10 --save /tmp/k1_mc$v.pt >> gpurun_out/${T}_k1_mc_ab.log 2>&1
  done
done
python -c "import torch; a=torch.load('/tmp/k1_mc0.pt'); b=torch.load('/tmp/k1_mc1.pt'); print('bit_identical', torch.equal(a,b))" >> gpurun_out/${T}_k1_mc_ab.log 2>&1
for v in 0 1; do
  STAR_K1_MC=$v timeout 300 python tools/phase1_bench.py --L 262144 --b 32768 --hq 64 --hkv 8 --iters 3 >> gpurun_out/${T}_k1_mc_ab.log 2>&1
done
tail -3 gpurun_out/${T}_k1_mc_tests.log; cat gpurun_out/${T}_k1_mc_ab.log
