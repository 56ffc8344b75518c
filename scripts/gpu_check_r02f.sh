# round-2 re-entry check (container re-created; library rebuilt from the last commit): smoke, GPU
# suite, headline bench (with e2e.batched), bench launch list
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_f.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_f.log 2>&1; tail -2 gpurun_out/smoke_f.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests_f.log 2>&1; tail -3 gpurun_out/gpu_tests_f.log
timeout 900 python bench.py > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err; tail -2 gpurun_out/bench_f.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_f.json 2> gpurun_out/bench_ref_f.err
