# occupancy caps (MGP_MINB_*: 8 CTAs of 256 threads per SM, 32 registers) for the cumsum passes, the
# prefix searches and the B-rule reduction: lb0 = ptxas default, lb1 = capped
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in lb0 lb1 lb0 lb1; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/lb_time.txt
  timeout 300 python scripts/mb/search_time.py >> gpurun_out/lb_time.txt 2>&1
  timeout 300 python scripts/kernel_table.py 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print([(r['kernel'][:22], r['ms']) for r in d['rows'] if any(k in r['kernel'] for k in ('weight_stats','cumsum','multinomial','systematic'))])" >> gpurun_out/lb_time.txt
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
