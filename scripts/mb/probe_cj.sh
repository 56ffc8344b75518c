# megores kernel: the accepted partner index carried instead of the round index (cj1) against cj0
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in cj0 cj1 cj0 cj1; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/cj_time.txt
  timeout 300 python scripts/mb/mego_time.py 2>&1 | grep megores >> gpurun_out/cj_time.txt
done
cp scripts/mb/libmgp_cj1.so paper_2109_13504_b200/libmgp.so
timeout 1200 python -m pytest tests/test_bracket_gpu.py tests/test_parity_gpu.py tests/test_reference_suite_gpu.py tests/test_reference_unmodified_gpu.py -q -x -p no:cacheprovider > gpurun_out/cj_tests.log 2>&1; tail -2 gpurun_out/cj_tests.log
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
