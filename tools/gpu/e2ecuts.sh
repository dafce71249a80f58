mkdir -p gpurun_out
O=gpurun_out/e2ecuts.log
{
timeout -s KILL 900 python -m pytest tests/test_kernels_gpu.py tests/test_pipeline_gpu.py -x -q 2>&1 | tail -3
timeout 100 python tools/k2_trace.py --rows 16384
timeout 100 python tools/decode_bench.py --rows 16384 --splits 0 --iters 200
for c in "0.5/0.5,0.75" "0.25,0.5/0.5,0.75,0.875" "0.125,0.25,0.5/0.5,0.75,0.875,0.9375" "0.0625,0.125,0.25,0.5/0.5,0.75,0.875,0.9375,0.96875"; do
  echo "CUTS=$c"
  STAR_E2E_CUTS=$c timeout -s KILL 600 python bench.py --no-cpu-baseline --no-sweep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print(d['value'], e['value'], e['ms_per_step'], e['augmented_layout']['value'])"
done
} > $O 2>&1
