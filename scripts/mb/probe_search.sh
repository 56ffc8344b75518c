# multinomial bucket table: K binary searches (old) vs one streaming pass (new); prefix tests
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in old new old new; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/search_time.txt
  timeout 300 python scripts/mb/search_time.py >> gpurun_out/search_time.txt 2>&1
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
timeout 1200 python -m pytest tests/test_prefix_gpu.py -q -x -p no:cacheprovider > gpurun_out/search_tests.log 2>&1; tail -3 gpurun_out/search_tests.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/search_launches.csv python scripts/mb/search_time.py > /dev/null 2>&1
