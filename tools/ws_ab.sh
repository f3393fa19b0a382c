#!/bin/bash
# A/B: two-shot all_reduce warp-specialized (1) vs CTA roles (0) on N GPUs
N=$1
for k in 1 0; do
  MCRDL_AR_KERNEL=$k python -m torch.distributed.run --nnodes 1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29571 -m paper_2303_08374_b200.tuner --ops all_reduce \
    --sizes 4M,16M,64M,256M,1G --iters 6 --warmup 2 --algorithms two_shot 2>/dev/null | grep "^all_reduce" | \
    awk -v k=$k -F, '{printf "ws=%s bytes=%s median=%sus busbw=%s\n", k, $3, $5, $7}'
done
