# round-2 evidence: compute-sanitizer over every product kernel, ncu launch list + full captures
TAG=${1:-r02}
mkdir -p gpurun_out
export STAR_EXCHANGE_TIMEOUT_S=600
# memcheck / initcheck over the product configuration; racecheck / synccheck run CTAs one at
# a time, so they take --serial (one split per group: no CTA spin-waits on another)
for tool in memcheck initcheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py \
    > gpurun_out/${TAG}_sanitize_${tool}.log 2>&1
  echo "exit=$?" >> gpurun_out/${TAG}_sanitize_${tool}.log
done
for tool in racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py --serial \
    > gpurun_out/${TAG}_sanitize_${tool}_serial.log 2>&1
  echo "exit=$?" >> gpurun_out/${TAG}_sanitize_${tool}_serial.log
done
unset STAR_EXCHANGE_TIMEOUT_S
bash tools_profile.sh ${TAG} > gpurun_out/${TAG}_profile.log 2>&1
