# compute-sanitizer over every product kernel (tools/sanitize_cases.py).  Usage: sanitize.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
export STAR_EXCHANGE_TIMEOUT_S=600
for tool in memcheck initcheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py \
    > gpurun_out/${TAG}_sanitize_${tool}.log 2>&1
  echo "exit=$?" >> gpurun_out/${TAG}_sanitize_${tool}.log
done
# racecheck / synccheck run CTAs one at a time: one split per group (--serial)
for tool in racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py --serial \
    > gpurun_out/${TAG}_sanitize_${tool}_serial.log 2>&1
  echo "exit=$?" >> gpurun_out/${TAG}_sanitize_${tool}_serial.log
done
