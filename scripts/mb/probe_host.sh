# host entry: chunk kernels on one stream (h1) vs alternating between two (h2); host-path tests
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in h1 h2 h1 h2; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/host_time.txt
  timeout 600 python scripts/mb/host_time.py >> gpurun_out/host_time.txt 2>&1
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_c_host_gpu.py tests/test_hygiene_gpu.py tests/test_prefix_gpu.py tests/test_reference_unmodified_gpu.py -q -p no:cacheprovider > gpurun_out/host_tests.log 2>&1; tail -3 gpurun_out/host_tests.log
