# compute-sanitizer over the all-kernels workload at the last code (incl. the megores brackets' re-runs)
set -x
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck initcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitizer/r02e_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer/rc_r02e.txt
done
