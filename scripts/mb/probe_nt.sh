# staging copies with streaming stores (nt1) against memcpy (nt0): pageable host-entry paths
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in nt0 nt1 nt0 nt1 nt0 nt1; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/nt_time.txt
  MGP_HOST_TRACE=1 timeout 300 python scripts/mb/dropin_breakdown.py 2>/tmp/tr_$v.txt | grep "host entry, pageable\|drop-in\|WeightVector" >> gpurun_out/nt_time.txt
  grep "staged_d2h" /tmp/tr_$v.txt | tail -2 | cut -c1-160 >> gpurun_out/nt_time.txt
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
timeout 900 python -m pytest tests/test_batch_gpu.py tests/test_c_host_gpu.py tests/test_parity_gpu.py tests/test_hygiene_gpu.py -q -x -p no:cacheprovider > gpurun_out/nt_tests.log 2>&1; tail -2 gpurun_out/nt_tests.log
