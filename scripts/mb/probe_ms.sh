# multinomial / systematic searches as programmatic dependents (ms1) against plain launches (ms0)
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in ms0 ms1 ms0 ms1; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/ms_time.txt
  timeout 300 python scripts/mb/search_ab.py >> gpurun_out/ms_time.txt 2>&1
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
timeout 1200 python -m pytest tests/test_prefix_gpu.py tests/test_reference_suite_gpu.py -q -x -p no:cacheprovider > gpurun_out/ms_tests.log 2>&1; tail -2 gpurun_out/ms_tests.log
