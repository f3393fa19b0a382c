#!/bin/bash
# two_shot all_reduce: all-gather by push (reducers store into peers) vs pull
# (gatherers read peers' reduced segments), with/without TMA senders, on N GPUs
N=$1
for cfg in "0 1" "1 1" "0 0" "1 0"; do
  set -- $cfg
  MCRDL_AR_AG_PULL=$1 MCRDL_AR_TMA=$2 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29545 -m paper_2303_08374_b200.tuner --ops all_reduce \
    --sizes 16M,64M,256M,1G --iters 8 --warmup 3 --algorithms two_shot 2>/dev/null | grep "^all_reduce" | \
    awk -v a=$1 -v t=$2 -F, '{printf "pull=%s tma=%s bytes=%s median=%sus busbw=%s\n", a, t, $3, $5, $7}'
done
