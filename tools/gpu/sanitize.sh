# compute-sanitizer over every product kernel (small shapes).  Usage: bash tools/gpu/sanitize.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py \
    > gpurun_out/${TAG}_sanitize_${tool}.log 2>&1
  echo "exit=$?" >> gpurun_out/${TAG}_sanitize_${tool}.log
done
