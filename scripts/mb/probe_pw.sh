# B-rule reduction: k_pw_final as a programmatic dependent of the chunk pass (pw1) against plain launches (pw0):
# weight-stats time and the bench step
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in pw0 pw1 pw0 pw1; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/pw_time.txt
  timeout 300 python scripts/kernel_table.py 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print([ (r['kernel'][:20], r['ms']) for r in d['rows'] if 'weight_stats' in r['kernel'] or 'quality' in r['kernel']])" >> gpurun_out/pw_time.txt
  timeout 300 python bench.py --no-cpu-baseline --quality-runs 0 --no-e2e --no-config5 --no-probe 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('step', round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms'],4))" >> gpurun_out/pw_time.txt
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_reference_suite_gpu.py tests/test_pfilter_gpu.py -q -x -p no:cacheprovider > gpurun_out/pw_tests.log 2>&1; tail -2 gpurun_out/pw_tests.log
