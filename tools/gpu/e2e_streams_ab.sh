# host-buffer pipeline: two compute streams (alternate blocks) vs one (STAR_E2E_COMP1=1);
# pipeline parity tests, then the bench's e2e number, alternating.  Usage: TAG
T=${1:-r02aa}
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_pipeline_gpu.py -m gpu -q > gpurun_out/${T}_pipeline_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pipeline_tests.log
for i in 1 2; do
  for v in 1 0; do
    STAR_E2E_COMP1=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-sweep 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('COMP1=$v', 'value', round(d['value']), 'e2e', round(d['e2e']['value']), 'e2e_ms', round(d['e2e']['ms_per_step'],2), 'ms', round(d['ms_per_step'],2), 'mhz', d['clocks']['sm_mhz'], 'match', d['e2e'].get('matches_device_path'))" >> gpurun_out/${T}_e2e_streams_ab.log
  done
done
tail -2 gpurun_out/${T}_pipeline_tests.log; cat gpurun_out/${T}_e2e_streams_ab.log
