# the megores bracket's accept test on subnormal weights: lenient (hi <= wj, HEAD) vs strict (hi < wj)
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in lenient strict; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/strict_tests.log
  timeout 900 python -m pytest tests/test_bracket_gpu.py -q -p no:cacheprovider >> gpurun_out/strict_tests.log 2>&1
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
true
true
