# A/B: bench kernel time with two builds of libmgp.so on the same box (alternating)
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_new.so
for r in 1 2; do
  for lib in scripts/mb/libmgp_head.so /tmp/libmgp_new.so; do
    cp $lib paper_2109_13504_b200/libmgp.so
    echo -n "$lib "; timeout 300 python bench.py --no-cpu-baseline --quality-runs 0 --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['roofline']['kernel_ms'])"
  done
done
cp /tmp/libmgp_new.so paper_2109_13504_b200/libmgp.so
