mkdir -p gpurun_out
for r in 0 1 2; do echo "REL=$r"; STAR_EXCHANGE_REL=$r timeout -s KILL 200 python tools/exchange_bench.py; done > gpurun_out/exb2.log 2>&1
STAR_EXCHANGE_REL=1 timeout -s KILL 300 ncu --set full --clock-control none -k regex:exchange_push -s 20 -c 1 -o gpurun_out/push_rel1 -f python tools/exchange_bench.py --rows 16384 > /dev/null 2>&1
