# one GPU call: tests, bench (headline), ncu launch list of the bench command, ncu full on the top kernel
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --quality-runs 0 --no-e2e > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_megopolis -s 1 -c 1 -o gpurun_out/prof_philox \
    python scripts/prof_step.py --steps 2 --rng philox > gpurun_out/ncu_philox.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_megopolis -s 1 -c 1 -o gpurun_out/prof_megores \
    python scripts/prof_step.py --steps 2 --rng megores > gpurun_out/ncu_megores.log 2>&1
ls gpurun_out
timeout 600 python scripts/kernel_table.py > gpurun_out/kernel_table.json 2> gpurun_out/kernel_table.err
