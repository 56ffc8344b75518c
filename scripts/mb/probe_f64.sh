# megores on float64 weights: bracketed (new) vs exact float64 path (old); parity tests
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in f64old f64new; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/f64_time.txt
  timeout 600 python scripts/mb/mego_time.py >> gpurun_out/f64_time.txt 2>&1
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_reference_suite_gpu.py tests/test_reference_unmodified_gpu.py tests/test_ipc_gpu.py -q -p no:cacheprovider > gpurun_out/f64_tests.log 2>&1; tail -3 gpurun_out/f64_tests.log
