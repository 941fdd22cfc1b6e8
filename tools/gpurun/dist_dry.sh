#!/bin/bash
# The torchrun branch of bench.py on a one-GPU box: 2 ranks share the GPU over gloo
# (a code-path check: shard, barrier, max-over-ranks timing, rank-ordered aggregate gather,
# cpu_baseline on rank 0 at N > 1) - not a scaling number.
mkdir -p gpurun_out
for cfg in c3 c2; do
  ALERT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --config $cfg --steps 2 --warmup 3 > gpurun_out/dist2_$cfg.json 2> gpurun_out/dist2_$cfg.err
  echo "$cfg rc=$?"; tail -1 gpurun_out/dist2_$cfg.json | cut -c1-300
done
ALERT_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/dist2_ref.json 2> gpurun_out/dist2_ref.err
echo "ref rc=$?"; tail -1 gpurun_out/dist2_ref.json | cut -c1-200
