# queued histogram's scatter kernel: register caps (CTAs per SM) and CTA shapes
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in 512_16_3 512_16_4 512_8_4 256_16_8 384_16_4 512_16_3; do
  cp scripts/mb/libmgp_oq_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/oq_time.txt
  timeout 300 python scripts/mb/offspring_time.py 2>&1 | grep "mode 0" >> gpurun_out/oq_time.txt
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
