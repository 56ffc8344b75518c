# megores half-split (4 particles per thread) A/B against one particle per thread; parity tests
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in mh0 mh1 mh0 mh1; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/mh_time.txt
  timeout 300 python scripts/mb/mego_time.py >> gpurun_out/mh_time.txt 2>&1
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_reference_suite_gpu.py tests/test_ipc_gpu.py -q -x -p no:cacheprovider > gpurun_out/mh_tests.log 2>&1; tail -3 gpurun_out/mh_tests.log
