# queued offspring histogram: A/B of (threads, ancestors per thread, CTAs per SM) builds; tests on the default
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in 512_16_1_0_2 hist4 512_16_1_0_2 hist4; do
  cp scripts/mb/libmgp_offq_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/offq2_time.txt
  timeout 300 python scripts/mb/offspring_time.py >> gpurun_out/offq2_time.txt 2>&1
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
timeout 900 python -m pytest tests/test_offspring_gpu.py -q -p no:cacheprovider > gpurun_out/offq2_tests.log 2>&1; tail -3 gpurun_out/offq2_tests.log
