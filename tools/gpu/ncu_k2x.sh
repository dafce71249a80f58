mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:phase2_mma -s 5 -c 1 -o gpurun_out/r01j_k2_16k -f python tools/decode_bench.py --rows 16384 --splits 0 --iters 10 > gpurun_out/ncu_k2x.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:phase2_mma -s 5 -c 1 -o gpurun_out/r01j_k2x_16k -f python tools/exchange_once.py 16384 >> gpurun_out/ncu_k2x.log 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"phase2_mma|exchange" -c 40 --csv --log-file gpurun_out/r01j_k2x_launches.csv python tools/exchange_once.py 131072 >> gpurun_out/ncu_k2x.log 2>&1
