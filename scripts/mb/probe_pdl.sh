# queued offspring histogram: programmatic dependent launch of k_offq_hist / k_offq_overflow (pdl1),
# plus k_offq_zero ahead of a PDL-launched scatter (pdz1), against plain stream order (pdl0)
# then the offspring and parity tests on pdz1
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in pdl0 pdl1 pdz1 pdl0 pdl1 pdz1; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/pdz_time.txt
  timeout 300 python scripts/mb/offspring_time.py 2>&1 | grep "mode 0" >> gpurun_out/pdz_time.txt
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
timeout 900 python -m pytest tests/test_offspring_gpu.py tests/test_parity_gpu.py -q -x -p no:cacheprovider > gpurun_out/pdz_tests.log 2>&1; tail -2 gpurun_out/pdz_tests.log
