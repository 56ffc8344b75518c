# batch host entry: the last job run in particle chunks with per-chunk downloads (lc1) against one launch (lc0)
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in lc0 lc1 lc0 lc1; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/lc_time.txt
  timeout 300 python scripts/mb/batch_time.py >> gpurun_out/lc_time.txt 2>&1
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
timeout 900 python -m pytest tests/test_batch_gpu.py tests/test_c_host_gpu.py tests/test_parity_gpu.py -q -x -p no:cacheprovider > gpurun_out/lc_tests.log 2>&1; tail -2 gpurun_out/lc_tests.log
