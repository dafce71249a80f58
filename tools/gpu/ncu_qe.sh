mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:phase2_qe -s 3 -c 1 -o gpurun_out/r01l_k2q -f env QB_ROWS=131072 QB_LQ=32 python tools/query_bench.py > gpurun_out/ncu_qe.log 2>&1
