# A/B: offspring histogram, int64 atomics (libmgp_off64.so) vs int32 in L2 + widen (current build)
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_new.so
for r in 1 2; do
  for lib in scripts/mb/libmgp_off64.so /tmp/libmgp_new.so; do
    cp $lib paper_2109_13504_b200/libmgp.so
    echo -n "$lib "; timeout 300 python scripts/kernel_table.py 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print([(r['kernel'], r['ms']) for r in d['rows'] if 'offspring' in r['kernel'] or 'quality' in r['kernel']])"
  done
done
cp /tmp/libmgp_new.so paper_2109_13504_b200/libmgp.so
