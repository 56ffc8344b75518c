# headline Philox kernel: float64 product (pf0) vs float32 bracket + exact re-run (pf1, and capped
# at 12 / 16 CTAs per SM: pfb12, pfb16); CUDA-event times + ancestor shas (scripts/mb/mego_time.py),
# then the bracket / parity suites on the bracket build
set -x
mkdir -p gpurun_out
cp paper_2109_13504_b200/libmgp.so /tmp/libmgp_keep.so
for v in pf0 pf1 pfb12 pfb16 pf0 pf1 pfb12 pfb16; do
  cp scripts/mb/libmgp_$v.so paper_2109_13504_b200/libmgp.so
  echo "== $v" >> gpurun_out/pf_time.txt
  timeout 300 python scripts/mb/mego_time.py >> gpurun_out/pf_time.txt 2>&1
done
cp /tmp/libmgp_keep.so paper_2109_13504_b200/libmgp.so
timeout 1200 python -m pytest tests/test_bracket_gpu.py tests/test_parity_gpu.py tests/test_reference_suite_gpu.py tests/test_ipc_gpu.py -q -x -p no:cacheprovider > gpurun_out/pf_tests.log 2>&1; tail -3 gpurun_out/pf_tests.log
