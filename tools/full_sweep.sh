#!/bin/bash
# Full per-op sweep with the NCCL comparator at N GPUs (run on the GPU box).
# usage: tools/full_sweep.sh N TAG
N=$1; TAG=$2
S=8,64,512,4K,32K,256K,1M,4M,16M,64M,256M,1G
for op in all_reduce all_to_allv all_gatherv bcast send; do
  timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29561 -m paper_2303_08374_b200.tuner --ops $op --sizes $S --iters 10 --warmup 3 \
    --nccl 2>/dev/null | grep -E "^$op"
done > gpurun_out/full_sweep_${TAG}.csv
echo "rows=$(wc -l < gpurun_out/full_sweep_${TAG}.csv)"
