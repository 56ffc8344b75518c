# round-2 final call (after the madc key add and the queued offspring histogram): smoke, GPU suite,
# headline bench, ncu captures of the Megopolis kernels (both streams) and the queued histogram's
# kernels, bench launch list, issue block, kernel table, compute-sanitizer over the all-kernels workload.
set -x
mkdir -p gpurun_out/sanitizer
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -2 gpurun_out/bench_final.err
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_megopolis -s 1 -c 1 -o gpurun_out/prof_philox -f python scripts/prof_step.py --steps 2 --rng philox > gpurun_out/ncu_philox.log 2>&1
$NCU -k regex:k_megopolis -s 1 -c 1 -o gpurun_out/prof_megores -f python scripts/prof_step.py --steps 2 --rng megores > gpurun_out/ncu_megores.log 2>&1
$NCU -k regex:k_megopolis -s 1 -c 1 -o gpurun_out/prof_philox_2p28 -f python scripts/prof_step.py --steps 2 --rng philox --n 268435456 > gpurun_out/ncu_philox_2p28.log 2>&1
$NCU -k regex:k_offq_scatter -s 2 -c 1 -o gpurun_out/prof_offq_scatter -f python scripts/mb/offspring_time.py > gpurun_out/ncu_offq.log 2>&1
$NCU -k regex:k_offq_hist -s 2 -c 1 -o gpurun_out/prof_offq_hist -f python scripts/mb/offspring_time.py >> gpurun_out/ncu_offq.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --quality-runs 0 --no-e2e --no-config5 --no-probe > gpurun_out/bench_under_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/offq_launches.csv python scripts/mb/offspring_time.py > /dev/null 2>&1
python scripts/issue_block.py philox@16777216@354=gpurun_out/prof_philox.ncu-rep megores@16777216@354=gpurun_out/prof_megores.ncu-rep \
    philox@268435456@354=gpurun_out/prof_philox_2p28.ncu-rep > gpurun_out/megopolis_issue.json 2> gpurun_out/issue_block.err
for r in philox megores philox_2p28 offq_scatter offq_hist; do python scripts/ncu_summary.py gpurun_out/prof_$r.ncu-rep "$r" > gpurun_out/sum_$r.txt; done
for r in philox megores offq_scatter; do ncu -i gpurun_out/prof_$r.ncu-rep --page source --csv > gpurun_out/src_$r.csv 2>/dev/null; done
rm -f gpurun_out/prof_*.ncu-rep
timeout 600 python scripts/kernel_table.py > gpurun_out/kernel_table.json 2> gpurun_out/kernel_table.err
timeout 300 python scripts/mb/mego_time.py > gpurun_out/mego_time.txt 2>&1
timeout 300 python scripts/mb/offspring_time.py > gpurun_out/offspring_time.txt 2>&1
for tool in memcheck racecheck initcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitizer/r02d_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer/rc_r02d.txt
done
du -sh gpurun_out
