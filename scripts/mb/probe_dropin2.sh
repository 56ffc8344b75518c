# drop-in call shape (pageable numpy in and out) at the session's start vs end library, same box
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in start end start end; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/dropin2.txt
  MGP_PINNED_OUTPUT=0 timeout 300 python scripts/mb/dropin_time.py 2>&1 | head -2 >> gpurun_out/dropin2.txt
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
