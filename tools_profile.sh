#!/bin/bash
# ncu evidence for the bench kernels (run under gpurun; single GPU).  Usage: tools_profile.sh TAG
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_launches_stdout.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:phase1_tc -s 3 -c 1 -o gpurun_out/${TAG}_k1 -f $B > gpurun_out/${TAG}_k1_stdout.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:phase2_mma -s 20 -c 1 -o gpurun_out/${TAG}_k2 -f $B > gpurun_out/${TAG}_k2_stdout.log 2>&1
ls -la gpurun_out
