# queued offspring histogram: correctness tests, A/B timing of the three modes, launch list
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_offspring_gpu.py -q -p no:cacheprovider > gpurun_out/offq_tests.log 2>&1; tail -3 gpurun_out/offq_tests.log
timeout 300 python scripts/mb/offspring_time.py > gpurun_out/offq_time.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/offq_launches.csv python scripts/mb/offspring_time.py > /dev/null 2>&1
