# ncu --set full of the exact cumsum's streaming kernels (third call) + summaries
mkdir -p gpurun_out
for k in k_px_aggregate k_px_materialize k_px_chunk_sum; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k python scripts/mb/cumsum_launches.py > /dev/null 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_$k.ncu-rep "$k" > gpurun_out/sum_$k.txt
  ncu -i gpurun_out/prof_$k.ncu-rep --page details --csv 2>/dev/null | grep -E '"Achieved Occupancy"|"Theoretical Occupancy"|"Registers Per Thread"|"Block Limit' > gpurun_out/occ_$k.txt
done
timeout 300 python scripts/mb/cumsum_time.py
