# exact cumsum: k_px_resolve / k_px_materialize as programmatic dependents (px1), plus the zeroing folded into k_px_chunk_sum and k_px_aggregate as a dependent of the scan (px2), against plain launches (px0)
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in px0 px1 px2 px0 px1 px2; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/pxpdl2_time.txt
  timeout 300 python scripts/mb/cumsum_time.py >> gpurun_out/pxpdl2_time.txt 2>&1
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
timeout 1200 python -m pytest tests/test_prefix_gpu.py tests/test_parity_gpu.py tests/test_reference_suite_gpu.py -q -x -p no:cacheprovider > gpurun_out/pxpdl2_tests.log 2>&1; tail -2 gpurun_out/pxpdl2_tests.log
