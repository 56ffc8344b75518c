set -x
mkdir -p gpurun_out
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; tail -2 gpurun_out/ref.err; cat gpurun_out/ref.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline --quality-runs 0 > gpurun_out/tr.json 2> gpurun_out/tr.err; tail -3 gpurun_out/tr.err; cat gpurun_out/tr.json | tail -1 | cut -c1-400
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29556 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/trref.json 2>&1; tail -1 gpurun_out/trref.json | cut -c1-300
