# round-2 profiling call: NCCL tests, ncu captures of the megopolis kernels (2^24 both streams,
# 2^28 philox), stale re-profiles (px_resolve, weight stats), the bench launch list, summaries.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_nccl_gpu.py > gpurun_out/nccl_tests.log 2>&1; tail -3 gpurun_out/nccl_tests.log
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_megopolis -s 1 -c 1 -o gpurun_out/prof_philox -f python scripts/prof_step.py --steps 2 --rng philox > gpurun_out/ncu_philox.log 2>&1
$NCU -k regex:k_megopolis -s 1 -c 1 -o gpurun_out/prof_megores -f python scripts/prof_step.py --steps 2 --rng megores > gpurun_out/ncu_megores.log 2>&1
$NCU -k regex:k_megopolis -s 1 -c 1 -o gpurun_out/prof_philox_2p28 -f python scripts/prof_step.py --steps 2 --rng philox --n 268435456 > gpurun_out/ncu_philox_2p28.log 2>&1
$NCU -k regex:k_px_resolve -s 0 -c 1 -o gpurun_out/prof_px_resolve -f python scripts/prof_step.py --steps 1 --kind multinomial > gpurun_out/ncu_px.log 2>&1
$NCU -k regex:k_pw_chunks -s 1 -c 1 -o gpurun_out/prof_stats -f python scripts/prof_step.py --steps 2 > gpurun_out/ncu_stats.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --quality-runs 0 --no-e2e --no-config5 --no-probe > gpurun_out/bench_under_ncu.log 2>&1
python scripts/issue_block.py philox@16777216@354=gpurun_out/prof_philox.ncu-rep megores@16777216@354=gpurun_out/prof_megores.ncu-rep \
    philox@268435456@354=gpurun_out/prof_philox_2p28.ncu-rep > gpurun_out/megopolis_issue.json 2> gpurun_out/issue_block.err
for r in philox megores philox_2p28 px_resolve stats; do python scripts/ncu_summary.py gpurun_out/prof_$r.ncu-rep "$r" > gpurun_out/sum_$r.txt; done
ls -la gpurun_out
# keep the merge-back under 64 MiB: raw CSV pages for everything, one report file
for r in philox megores philox_2p28 px_resolve stats; do ncu -i gpurun_out/prof_$r.ncu-rep --page raw --csv > gpurun_out/raw_$r.csv 2>/dev/null; done
ncu -i gpurun_out/prof_philox.ncu-rep --page source --csv > gpurun_out/src_philox.csv 2>/dev/null
ncu -i gpurun_out/prof_megores.ncu-rep --page source --csv > gpurun_out/src_megores.csv 2>/dev/null
rm -f gpurun_out/prof_megores.ncu-rep gpurun_out/prof_philox_2p28.ncu-rep gpurun_out/prof_px_resolve.ncu-rep gpurun_out/prof_stats.ncu-rep
cat gpurun_out/nccl_tests.log | tail -5
du -sh gpurun_out
