# host entry: the last chunk cut into a half and two quarters for page-locked outputs (ts2; ts1 also for pageable ones) against equal chunks (ts0)
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in ts0 ts2 ts0 ts2; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/ts2_time.txt
  timeout 300 python scripts/mb/host_time.py >> gpurun_out/ts2_time.txt 2>&1
  timeout 300 python scripts/mb/dropin_breakdown.py 2>&1 | grep "host entry\|drop-in" >> gpurun_out/ts2_time.txt
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
timeout 1200 python -m pytest tests/test_batch_gpu.py tests/test_c_host_gpu.py tests/test_parity_gpu.py -q -x -p no:cacheprovider > gpurun_out/ts2_tests.log 2>&1; tail -2 gpurun_out/ts2_tests.log
