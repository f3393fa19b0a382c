#!/bin/bash
# all_reduce two_shot at 64M/256M/1G for several (GPMAX, CHUNK_KB) settings on N GPUs
N=$1
for cfg in "98 256" "74 256" "49 256" "98 128" "98 512" "98 1024" "74 512" "64 1024"; do
  set -- $cfg
  MCRDL_AR_GPMAX=$1 MCRDL_AR_CHUNK_KB=$2 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29541 -m paper_2303_08374_b200.tuner --ops all_reduce \
    --sizes 64M,256M,1G --iters 6 --warmup 2 --algorithms two_shot 2>/dev/null | grep "^all_reduce" | \
    awk -v g=$1 -v c=$2 -F, '{printf "gp=%s chunk=%sK bytes=%s median=%sus busbw=%s\n", g, c, $3, $5, $7}'
done
