#!/bin/bash
# Round-end measurement set (run on the GPU box): per-op sweeps with NCCL at
# p=2/4, bf16 all_reduce, and all_reduce on symmetric tensors.
S=8,512,4K,32K,256K,1M,4M,16M,64M,256M,1G
for N in 4 2; do
  DEV=$(seq -s, 0 $((N-1)))
  for op in all_reduce all_to_allv all_gatherv bcast send; do
    CUDA_VISIBLE_DEVICES=$DEV timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops $op --sizes $S \
      --iters 10 --warmup 3 --nccl 2>/dev/null | grep -E "^$op"
  done > gpurun_out/final_sweep_p$N.csv
  CUDA_VISIBLE_DEVICES=$DEV timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops all_reduce \
    --sizes $S --iters 10 --warmup 3 --dtype bf16 --nccl 2>/dev/null | grep -E "^all_reduce" \
    > gpurun_out/final_sweep_bf16_p$N.csv
  CUDA_VISIBLE_DEVICES=$DEV timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops all_reduce \
    --sizes 1M,4M,16M,64M,256M,1G --iters 10 --warmup 3 --symm --algorithms auto 2>/dev/null \
    | grep -E "^all_reduce" > gpurun_out/final_symm_p$N.csv
  echo "p$N rows: $(wc -l < gpurun_out/final_sweep_p$N.csv) bf16 $(wc -l < gpurun_out/final_sweep_bf16_p$N.csv) symm $(wc -l < gpurun_out/final_symm_p$N.csv)"
done
