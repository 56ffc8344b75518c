# ncu --set full of the queued histogram's two kernels
set -x
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_offq_scatter -s 2 -c 1 -o gpurun_out/prof_offq_scatter -f python scripts/mb/offspring_time.py > gpurun_out/ncu_offq.log 2>&1
$NCU -k regex:k_offq_hist -s 2 -c 1 -o gpurun_out/prof_offq_hist -f python scripts/mb/offspring_time.py >> gpurun_out/ncu_offq.log 2>&1
for r in offq_scatter offq_hist; do python scripts/ncu_summary.py gpurun_out/prof_$r.ncu-rep "$r" > gpurun_out/sum_$r.txt; ncu -i gpurun_out/prof_$r.ncu-rep --page raw --csv > gpurun_out/raw_$r.csv 2>/dev/null; ncu -i gpurun_out/prof_$r.ncu-rep --page source --csv > gpurun_out/src_$r.csv 2>/dev/null; done
rm -f gpurun_out/prof_*.ncu-rep
