# exact cumsum / prefix resamplers: tests, initcheck + memcheck over the sanitizer workload, timing
mkdir -p gpurun_out/sanitizer
timeout 900 python -m pytest tests -x -q -m gpu -k "prefix or cumsum or multinomial or systematic" 2>&1 | tail -2
for tool in initcheck memcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitizer/r02c_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -1 gpurun_out/sanitizer/r02c_$tool.txt
done
timeout 300 python scripts/mb/cumsum_time.py
timeout 300 python scripts/mb/search_time.py
