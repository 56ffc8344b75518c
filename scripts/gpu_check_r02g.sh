# after the host pool sizing fix (half the hardware threads, at most 8): GPU suite, drop-in
# breakdown, headline bench
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests_g.log 2>&1; tail -3 gpurun_out/gpu_tests_g.log
timeout 300 python scripts/mb/dropin_breakdown.py > gpurun_out/dropin_bd_g.txt 2>&1
timeout 300 python scripts/mb/dropin_breakdown2.py > gpurun_out/dropin_bd2_g.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; tail -2 gpurun_out/bench_g.err
