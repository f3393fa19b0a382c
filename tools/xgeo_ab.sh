#!/bin/bash
# Exchange geometry A/B: bytes of a pair per serving CTA (MCRDL_X_PAIR_KB) x
# minimum flag chunk (MCRDL_X_CHUNK_KB), all_to_allv on N GPUs.
N=$1
for P in 32 64 128; do
  for C in 64 128 256; do
    MCRDL_X_PAIR_KB=$P MCRDL_X_CHUNK_KB=$C timeout 300 python -m torch.distributed.run --nnodes 1 \
      --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29581 -m paper_2303_08374_b200.tuner \
      --ops all_to_allv --sizes 4M,16M,64M,256M --iters 20 --warmup 3 --algorithms direct_write \
      2>/dev/null | grep "^all_to_allv" | sed "s/^/pair=${P}K chunk=${C}K /"
  done
done
