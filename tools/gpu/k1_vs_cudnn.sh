# ncu side by side: our K1 vs cuDNN SDPA on one 32K causal block; K1 clock64 trace
TAG=${1:-r02}
mkdir -p gpurun_out
make -C paper_2411_17116_b200/csrc trace -j8 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_cudnn_launches.csv \
  python tools/k1_vs_cudnn.py cudnn 32768 3 > gpurun_out/${TAG}_cudnn_list.log 2>&1
KN=$(python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/${TAG}_cudnn_launches.csv")))
h=[i for i,r in enumerate(rows) if r and r[0]=="ID"][0]
hdr=rows[h]; ki=hdr.index("Kernel Name"); vi=hdr.index("Metric Value")
best=max(rows[h+1:], key=lambda r: float(r[vi].replace(",","")) if len(r)>vi else 0)
print(best[ki].split("(")[0].split("<")[0].strip().split(" ")[-1])
PY
)
echo "cudnn kernel: $KN" > gpurun_out/${TAG}_cudnn_name.txt
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k "regex:$KN" -c 1 \
  -o gpurun_out/${TAG}_cudnn python tools/k1_vs_cudnn.py cudnn 32768 2 > gpurun_out/${TAG}_cudnn_ncu.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:phase1_tc -c 1 \
  -o gpurun_out/${TAG}_ours python tools/k1_vs_cudnn.py ours 32768 1 > gpurun_out/${TAG}_ours_ncu.log 2>&1
timeout -s KILL 300 python tools/k1_trace.py > gpurun_out/${TAG}_k1_trace.log 2>&1
