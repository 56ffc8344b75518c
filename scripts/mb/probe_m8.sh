# megores Megopolis and C1/C2 at eight 256-thread CTAs per SM (32 registers) vs ptxas's choice
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in m0 m8 m0 m8; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/m8_time.txt
  timeout 300 python scripts/mb/mego_time.py 2>&1 | grep "f32" >> gpurun_out/m8_time.txt
  timeout 600 python scripts/mb/c12_time.py 2>&1 | grep megores >> gpurun_out/m8_time.txt
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
