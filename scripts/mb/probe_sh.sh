# megores Megopolis: high-word right shifts of splitmix as IMAD.HI (FMA pipe) vs SHF (ALU pipe)
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in sh0 sh1 sh2 sh0 sh1 sh2; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/sh_time.txt
  timeout 300 python scripts/mb/mego_time.py 2>&1 | grep "megores  f32" >> gpurun_out/sh_time.txt
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
