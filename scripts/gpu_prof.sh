set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --quality-runs 0 --no-e2e > gpurun_out/bench_dbg.json 2>&1; tail -1 gpurun_out/bench_dbg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['step_breakdown_ms'], d['roofline']['kernel_ms'])"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/prof_step.py --steps 3 > /dev/null 2>&1
grep -v "^==" gpurun_out/launches.csv | tail -7 | cut -d, -f5,15-16
ncu --set full --clock-control none --import-source on -k regex:k_megopolis -s 1 -c 1 -o gpurun_out/prof_mego2 python scripts/prof_step.py --steps 2 > gpurun_out/ncu_mego2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_megopolis -s 1 -c 1 -o gpurun_out/prof_mego_philox python scripts/prof_step.py --steps 2 --rng philox > gpurun_out/ncu_mego3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pw_chunks -s 0 -c 1 -o gpurun_out/prof_stats2 python scripts/prof_step.py --steps 1 > gpurun_out/ncu_stats2.log 2>&1
ls gpurun_out
