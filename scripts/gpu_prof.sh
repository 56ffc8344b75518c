set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/prof_step.py --steps 3 > /dev/null 2>&1
tail -12 gpurun_out/launches.csv
ncu --set full --clock-control none --import-source on -k regex:k_megopolis -s 1 -c 1 -o gpurun_out/prof_mego python scripts/prof_step.py --steps 2 > gpurun_out/ncu_mego.log 2>&1
tail -3 gpurun_out/ncu_mego.log
ncu --set full --clock-control none --import-source on -k regex:k_metropolis -s 0 -c 1 -o gpurun_out/prof_metro python scripts/prof_step.py --steps 1 --kind metropolis > gpurun_out/ncu_metro.log 2>&1
tail -3 gpurun_out/ncu_metro.log
ncu --set full --clock-control none --import-source on -k regex:k_pw_chunks -s 0 -c 1 -o gpurun_out/prof_stats python scripts/prof_step.py --steps 1 > gpurun_out/ncu_stats.log 2>&1
ls -la gpurun_out
