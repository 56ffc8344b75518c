# the bench's N > 1 code path end to end on one GPU: 2 and 4 ranks on cuda:0 with gloo collectives
# (MGP_BENCH_LOOPBACK=1, test plumbing; the numbers are not multi-GPU numbers)
set -x
mkdir -p gpurun_out
for g in 2 4; do
  MGP_BENCH_LOOPBACK=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $g --master-addr 127.0.0.1 \
      --master-port 2953$g bench.py --gpus $g --steps 3 --warmup 3 --quality-runs 0 > gpurun_out/loopback_$g.json 2> gpurun_out/loopback_$g.err
  echo "rc=$?" >> gpurun_out/loopback_$g.err
done
