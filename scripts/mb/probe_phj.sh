# headline Philox kernel: the accepted partner index carried instead of the round index (phj1) vs phj0
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in phj0 phj1 phj0 phj1 phj0 phj1; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/phj_time.txt
  timeout 300 python scripts/mb/mego_time.py 2>&1 | grep "philox   f32" >> gpurun_out/phj_time.txt
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
