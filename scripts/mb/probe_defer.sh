# queued histogram: deferred queue reservations for K <= 4 * 512 (d4, 4-byte spill) vs K <= 2 * 512 (d2, no spill)
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in d4 d2 d4 d2; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/defer_time.txt
  timeout 300 python scripts/mb/offspring_time.py 2>&1 | grep "mode 0" >> gpurun_out/defer_time.txt
done
cp scripts/mb/libmgp_d2.so paper_2109_13504_b200/libmgp.so; timeout 900 python -m pytest tests/test_offspring_gpu.py -q -p no:cacheprovider > gpurun_out/defer_tests.log 2>&1; tail -2 gpurun_out/defer_tests.log
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
