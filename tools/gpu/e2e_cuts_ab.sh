# host-buffer pipeline fill / drain cut fractions (STAR_E2E_CUTS) with the two compute streams
T=${1:-r02ab}
mkdir -p gpurun_out
for i in 1 2; do
  for c in "0.5/0.5,0.75" "/" "0.25,0.5/0.5,0.75,0.875" "0.5/0.75" "0.25,0.5,0.75/0.5,0.75"; do
    STAR_E2E_CUTS=$c timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-sweep 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('CUTS=$c', 'e2e', round(d['e2e']['value']), 'e2e_ms', round(d['e2e']['ms_per_step'],2), 'ms', round(d['ms_per_step'],2), 'match', d['e2e'].get('matches_device_path'))" >> gpurun_out/${T}_e2e_cuts.log
  done
done
cat gpurun_out/${T}_e2e_cuts.log
