#!/bin/bash
# staged NVLS all_reduce: flag chunk x reducer CTAs (copiers/gatherers 16) on N GPUs
N=$1
for C in 128 256 512 1024; do for G in 24 32 48; do
  MCRDL_AR_CHUNK_KB=$C MCRDL_NVLS_GP=$G timeout 200 python -m torch.distributed.run --nnodes 1 \
    --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29583 -m paper_2303_08374_b200.tuner \
    --ops all_reduce --sizes 256M,1G --iters 8 --warmup 3 --algorithms nvls 2>/dev/null | \
    grep "^all_reduce" | sed "s/^/chunk=${C}K gp=$G /"
done; done
