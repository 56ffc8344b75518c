# round-2 last call (after the PDL launches of the cumsum / search / B-rule kernels, the megores
# partner-index carry and the host-entry tail split): smoke, GPU suite, bench, reference arm, kernel table, launch lists
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_y.log 2>&1; tail -2 gpurun_out/smoke_y.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests_y.log 2>&1; tail -3 gpurun_out/gpu_tests_y.log
timeout 900 python bench.py > gpurun_out/bench_y.json 2> gpurun_out/bench_y.err; tail -2 gpurun_out/bench_y.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_y.json 2> gpurun_out/bench_ref_y.err
timeout 600 python scripts/kernel_table.py > gpurun_out/kernel_table_y.json 2> gpurun_out/kernel_table_y.err
timeout 300 python scripts/mb/offspring_time.py > gpurun_out/offspring_time_y.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches_y.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --quality-runs 0 --no-e2e --no-config5 --no-probe > gpurun_out/bench_under_ncu_y.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/offq_launches_y.csv python scripts/mb/offspring_time.py > /dev/null 2>&1
