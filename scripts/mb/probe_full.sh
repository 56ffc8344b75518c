# full GPU suite + megopolis timing + offspring timing at the current build
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/full_tests.log 2>&1; tail -3 gpurun_out/full_tests.log
timeout 300 python scripts/mb/mego_time.py > gpurun_out/full_mego.txt 2>&1
timeout 300 python scripts/mb/offspring_time.py > gpurun_out/full_off.txt 2>&1
