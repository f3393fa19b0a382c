#!/bin/bash
# A/B: two-shot all_reduce with and without TMA senders on N GPUs
N=$1
for cfg in "2 64" "2 32" "0 0"; do
  set -- $cfg
  MCRDL_AR_TMA=$1 MCRDL_AR_TMA_CTAS=$2 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29551 -m paper_2303_08374_b200.tuner --ops all_reduce \
    --sizes 16M,64M,256M,1G --iters 6 --warmup 2 --algorithms two_shot 2>/dev/null | grep "^all_reduce" | \
    awk -v t=$1 -v g=$2 -F, '{printf "tma=%s ctas=%s bytes=%s median=%sus busbw=%s\n", t, g, $3, $5, $7}'
done
