# round-2 very last call (after the batch entry chunks its last job): smoke, GPU suite, bench, reference arm
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_x.log 2>&1; tail -2 gpurun_out/smoke_x.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests_x.log 2>&1; tail -3 gpurun_out/gpu_tests_x.log
timeout 900 python bench.py > gpurun_out/bench_x.json 2> gpurun_out/bench_x.err; tail -2 gpurun_out/bench_x.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_x.json 2> gpurun_out/bench_ref_x.err
