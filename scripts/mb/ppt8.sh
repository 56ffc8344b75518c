cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_default.so
cp scripts/mb/libmgp_p8.so paper_2109_13504_b200/libmgp.so
python scripts/kernel_table.py --reps 3 | python -c "
import json,sys; d=json.load(sys.stdin)
for r in d['rows'][:2]: print('PPT8', r['kernel'], r['ms'], r['frac_of_hbm'])"
cp /tmp/libmgp_default.so paper_2109_13504_b200/libmgp.so
