# compute-sanitizer over the small all-kernels workload (scripts/sanitize.py)
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck initcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitizer/r02_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer/rc.txt
done
