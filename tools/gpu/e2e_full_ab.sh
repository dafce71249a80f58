# the default bench command (as the driver runs it) with one vs two compute streams in the e2e pipeline
T=${1:-r02ad}
mkdir -p gpurun_out
for i in 1 2; do
  for v in 1 0; do
    STAR_E2E_COMP1=$v timeout 900 python bench.py 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('COMP1=$v', 'value', round(d['value']), 'e2e', round(d['e2e']['value']), 'e2e_ms', round(d['e2e']['ms_per_step'],2), 'ms', round(d['ms_per_step'],2), 'mhz', d['clocks']['sm_mhz'])" >> gpurun_out/${T}_e2e_full_ab.log
  done
done
cat gpurun_out/${T}_e2e_full_ab.log
