set -x
mkdir -p gpurun_out
timeout 600 python scripts/kernel_table.py > gpurun_out/kt_madc.json 2> gpurun_out/kt_madc.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/off_launches.csv python scripts/mb/offspring_time.py > gpurun_out/off_time_ncu.txt 2>&1
timeout 300 python scripts/mb/offspring_time.py > gpurun_out/off_time.txt 2>&1
