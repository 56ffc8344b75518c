# drop-in call shape with a page-locked result array; host-path tests
set -x
mkdir -p gpurun_out
timeout 600 python scripts/mb/dropin_time.py > gpurun_out/dropin_time.txt 2>&1
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_c_host_gpu.py tests/test_reference_unmodified_gpu.py tests/test_hygiene_gpu.py -q -p no:cacheprovider > gpurun_out/dropin_tests.log 2>&1; tail -3 gpurun_out/dropin_tests.log
