# exact cumsum: parity tests, timing (A/B vs HEAD build), resolver profile, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "prefix or cumsum or multinomial or systematic" 2>&1 | tail -3
timeout 300 python scripts/mb/cumsum_time.py
bash scripts/mb/px_prof.sh
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cumsum_f32_launches.csv python scripts/mb/cumsum_launches.py > /dev/null 2>&1
