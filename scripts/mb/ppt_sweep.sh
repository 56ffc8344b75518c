# time the Megopolis kernels with alternative particles-per-thread builds of libmgp.so
for lib in scripts/mb/libmgp_p4_m2.so scripts/mb/libmgp_p2_m2.so scripts/mb/libmgp_p4_m1.so; do
  cp $lib paper_2109_13504_b200/libmgp.so
  echo "== $lib"
  python scripts/kernel_table.py --reps 3 | python -c "
import json,sys; d=json.load(sys.stdin)
for r in d['rows'][:2]: print(r['kernel'], r['ms'], r['frac_of_hbm'])"
done
