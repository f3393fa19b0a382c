#!/bin/bash
# LL vs bulk thresholds: all_reduce (MCRDL_LL_MAX_BYTES) and per-pair exchange
# (MCRDL_LL_PAIR_BYTES) at 64K..4M on N GPUs
N=$1
for T in 65536 131072 262144; do
  MCRDL_LL_PAIR_BYTES=$T MCRDL_LL_MAX_BYTES=$T timeout 300 python -m torch.distributed.run --nnodes 1 \
    --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29577 -m paper_2303_08374_b200.tuner \
    --ops all_reduce,all_to_allv,all_gatherv,bcast --sizes 64K,128K,256K,512K,1M,2M,4M --iters 10 \
    --warmup 3 --algorithms one_shot,direct_write 2>/dev/null | grep -E "^(all|bcast)" | sed "s/^/T=$T /"
done
