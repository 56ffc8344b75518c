# headline Philox kernel A/B: float64 product (pf0) vs float32 bracket variants (pa0: bool
# ambiguity flags, chained hi; pc: hi from 1 + u23 + 2^-23, independent of lo)
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in pf0 pa0 pc pf0 pa0 pc; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/pf_time_b.txt
  timeout 300 python scripts/mb/mego_time.py 2>&1 | grep philox >> gpurun_out/pf_time_b.txt
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
