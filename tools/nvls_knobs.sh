#!/bin/bash
# all_reduce nvls at 64M/256M for several (FENCE, GPMAX, CHUNK_KB) settings on N GPUs
N=$1
for cfg in "0 8 256" "0 12 256" "0 16 256" "0 24 256" "0 32 256" "0 40 256" "0 16 128" "0 24 128" "0 16 512" "0 24 512"; do
  set -- $cfg
  MCRDL_NVLS_FENCE=$1 MCRDL_AR_GPMAX=$2 MCRDL_AR_CHUNK_KB=$3 python -m torch.distributed.run --nnodes 1 \
    --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29543 -m paper_2303_08374_b200.tuner \
    --ops all_reduce --sizes 64M,256M,1G --iters 6 --warmup 2 --algorithms nvls 2>/dev/null | grep "^all_reduce" | \
    awk -v f=$1 -v g=$2 -v c=$3 -F, '{printf "fence=%s gp=%s chunk=%sK bytes=%s median=%sus busbw=%s\n", f, g, c, $3, $5, $7}'
done
