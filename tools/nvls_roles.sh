#!/bin/bash
# NVLS all_reduce role widths (reducers GP, copiers GC, gatherers GG) on N GPUs
N=$1
for cfg in "32 32 32" "48 24 24" "48 16 16" "64 16 16" "32 16 16" "64 24 24" "40 20 20"; do
  set -- $cfg
  MCRDL_NVLS_GP=$1 MCRDL_NVLS_GC=$2 MCRDL_NVLS_GG=$3 python -m torch.distributed.run --nnodes 1 \
    --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29553 -m paper_2303_08374_b200.tuner \
    --ops all_reduce --sizes 64M,256M,1G --iters 8 --warmup 3 --algorithms nvls 2>/dev/null | \
    grep "^all_reduce" | awk -v a=$1 -v b=$2 -v c=$3 -F, \
    '{printf "gp=%s gc=%s gg=%s bytes=%s median=%sus busbw=%s\n", a, b, c, $3, $5, $7}'
done
