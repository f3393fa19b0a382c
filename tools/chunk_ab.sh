#!/bin/bash
# two-shot all_reduce chunk size (MCRDL_AR_CHUNK_KB) vs message size on N GPUs
N=$1
for C in 32 64 128 256; do
  MCRDL_AR_CHUNK_KB=$C timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29579 -m paper_2303_08374_b200.tuner --ops all_reduce \
    --sizes 4M,16M,64M,256M --iters 10 --warmup 3 --algorithms two_shot 2>/dev/null | \
    grep "^all_reduce" | sed "s/^/chunk=${C}K /"
done
