# host entry with pageable buffers against the page-locked staging slot size (4 / 8 / 16 MiB)
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in sl8 sl16 sl4 sl8 sl16 sl4; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/slot_time.txt
  MGP_HOST_TRACE=1 timeout 300 python scripts/mb/dropin_breakdown.py 2>/tmp/trace_$v.txt | grep "host entry, pageable\|drop-in" >> gpurun_out/slot_time.txt
  grep staged_h2d /tmp/trace_$v.txt | tail -3 >> gpurun_out/slot_time.txt
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
