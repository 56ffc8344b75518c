# round-2 closing refresh (after the 8-worker host pool and the PDL-launched queued histogram):
# smoke, GPU suite, headline bench, reference arm, kernel table, bench launch list, ncu --set full of
# the queued histogram's kernels and of the headline kernel
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_z.log 2>&1; tail -2 gpurun_out/smoke_z.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests_z.log 2>&1; tail -3 gpurun_out/gpu_tests_z.log
timeout 900 python bench.py > gpurun_out/bench_z.json 2> gpurun_out/bench_z.err; tail -2 gpurun_out/bench_z.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_z.json 2> gpurun_out/bench_ref_z.err
timeout 600 python scripts/kernel_table.py > gpurun_out/kernel_table_z.json 2> gpurun_out/kernel_table_z.err
timeout 300 python scripts/mb/offspring_time.py > gpurun_out/offspring_time_z.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches_z.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --quality-runs 0 --no-e2e --no-config5 --no-probe > gpurun_out/bench_under_ncu_z.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/offq_launches_z.csv python scripts/mb/offspring_time.py > /dev/null 2>&1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_offq_scatter -s 2 -c 1 -o gpurun_out/prof_offq_scatter -f python scripts/mb/offspring_time.py > gpurun_out/ncu_offq_z.log 2>&1
$NCU -k regex:k_offq_hist -s 2 -c 1 -o gpurun_out/prof_offq_hist -f python scripts/mb/offspring_time.py >> gpurun_out/ncu_offq_z.log 2>&1
$NCU -k regex:k_megopolis -s 1 -c 1 -o gpurun_out/prof_philox -f python scripts/prof_step.py --steps 2 --rng philox > gpurun_out/ncu_philox_z.log 2>&1
for r in offq_scatter offq_hist philox; do python scripts/ncu_summary.py gpurun_out/prof_$r.ncu-rep "$r" > gpurun_out/sum_z_$r.txt; done
rm -f gpurun_out/prof_*.ncu-rep
