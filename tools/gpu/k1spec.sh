mkdir -p gpurun_out
O=gpurun_out/k1spec.log
{
for r in 1 2; do
  STAR_K1_SPEC=0 timeout 300 python tools/phase1_bench.py --iters 5 --save /tmp/o0.pt
  STAR_K1_SPEC=1 timeout 300 python tools/phase1_bench.py --iters 5 --save /tmp/o1.pt
done
python -c "import torch; a=torch.load('/tmp/o0.pt'); b=torch.load('/tmp/o1.pt'); print('bit-exact', torch.equal(a,b), (a.float()-b.float()).abs().max().item())"
STAR_K1_SPEC=1 timeout 300 python tools/phase1_bench.py --L 262144 --b 32768 --hq 64 --iters 2
STAR_K1_SPEC=0 timeout 300 python tools/phase1_bench.py --L 262144 --b 32768 --hq 64 --iters 2
} > $O 2>&1
STAR_K1_SPEC=1 timeout 300 python tools/k1_trace.py >> $O 2>&1
STAR_K1_SPEC=0 timeout 300 python tools/k1_trace.py >> $O 2>&1
