# batch host entry: uploads/statistics on a highest-priority stream (bp1) against normal priority (bp0)
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in bp0 bp1 bp0 bp1; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/bp_time.txt
  timeout 300 python scripts/mb/batch_time.py >> gpurun_out/bp_time.txt 2>&1
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
timeout 900 python -m pytest tests/test_batch_gpu.py tests/test_c_host_gpu.py -q -x -p no:cacheprovider > gpurun_out/bp_tests.log 2>&1; tail -2 gpurun_out/bp_tests.log
