#!/bin/bash
# NVLS bcast at 16M/256M for several (CTAS, CHUNK_KB) settings on N GPUs
N=$1
for cfg in "74 256" "148 256" "32 256" "74 64" "74 1024" "148 128" "16 1024"; do
  set -- $cfg
  MCRDL_BCAST_CTAS=$1 MCRDL_BCAST_CHUNK_KB=$2 python -m torch.distributed.run --nnodes 1 \
    --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29551 -m paper_2303_08374_b200.tuner \
    --ops bcast --sizes 16M,256M --iters 8 --warmup 3 --algorithms nvls 2>/dev/null | grep "^bcast" | \
    awk -v g=$1 -v c=$2 -F, '{printf "ctas=%s chunk=%sK bytes=%s median=%sus busbw=%s\n", g, c, $3, $5, $7}'
done
