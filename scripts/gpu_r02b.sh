mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cumsum_f32_launches.csv python scripts/mb/cumsum_launches.py > /dev/null 2>&1
PREC=double ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cumsum_f64_launches.csv python scripts/mb/cumsum_launches.py > /dev/null 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "megores or parity or reference" 2>&1 | tail -3
timeout 300 python bench.py --rng megores --steps 10 --warmup 3 --no-cpu-baseline --quality-runs 0 --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('megores kernel_ms', d['roofline']['kernel_ms'], d['value'])"
