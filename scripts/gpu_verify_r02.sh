# re-entry check after a container restore: smoke, full GPU suite, headline bench
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_verify.json 2> gpurun_out/bench_verify.err; tail -2 gpurun_out/bench_verify.err
