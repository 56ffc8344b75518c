# refresh the ncu issue block (profiles/megopolis_issue.json) at the last code (megores kernel with
# the partner-index carry)
set -x
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_megopolis -s 1 -c 1 -o gpurun_out/prof_philox -f python scripts/prof_step.py --steps 2 --rng philox > gpurun_out/ncu_philox_v.log 2>&1
$NCU -k regex:k_megopolis -s 1 -c 1 -o gpurun_out/prof_megores -f python scripts/prof_step.py --steps 2 --rng megores > gpurun_out/ncu_megores_v.log 2>&1
$NCU -k regex:k_megopolis -s 1 -c 1 -o gpurun_out/prof_philox_2p28 -f python scripts/prof_step.py --steps 2 --rng philox --n 268435456 > gpurun_out/ncu_philox_2p28_v.log 2>&1
python scripts/issue_block.py philox@16777216@354=gpurun_out/prof_philox.ncu-rep megores@16777216@354=gpurun_out/prof_megores.ncu-rep \
    philox@268435456@354=gpurun_out/prof_philox_2p28.ncu-rep > gpurun_out/megopolis_issue_v.json 2> gpurun_out/issue_block_v.err
for r in philox megores philox_2p28; do python scripts/ncu_summary.py gpurun_out/prof_$r.ncu-rep "$r" > gpurun_out/sum_v_$r.txt; done
rm -f gpurun_out/prof_*.ncu-rep
