# megores splitmix: x * MIX1 in three instructions (IMAD.WIDE + 2 IMAD, mul3) against ptxas's four (mul0)
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in mul0 mul1 mul0 mul1; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/mul3_time.txt
  timeout 300 python scripts/mb/mego_time.py >> gpurun_out/mul3_time.txt 2>&1
  timeout 300 python scripts/mb/c12_time.py 2>&1 | grep megores >> gpurun_out/mul3_time.txt
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
