# round-2 last evidence refresh (after the C1/C2 megores bracket, the strict accept test and the
# two-stream host chunks): smoke, GPU suite, headline bench, kernel table, megores ncu issue block
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_final_d.json 2> gpurun_out/bench_final_d.err; tail -2 gpurun_out/bench_final_d.err
timeout 600 python scripts/kernel_table.py > gpurun_out/kernel_table_d.json 2> gpurun_out/kernel_table_d.err
timeout 600 python scripts/mb/host_time.py > gpurun_out/host_time_d.txt 2>&1
timeout 600 python scripts/mb/c12_time.py > gpurun_out/c12_time_d.txt 2>&1
