cd $GRAFT_REPO_ROOT
S=8,4K,32K,128K,256K
for N in 4 2; do
  DEV=$(seq -s, 0 $((N-1)))
  for LL in 262144 65536; do
    for op in all_reduce all_to_allv; do
      MCRDL_LL_MAX_BYTES=$LL MCRDL_LL_PAIR_BYTES=$LL CUDA_VISIBLE_DEVICES=$DEV timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N \
        --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops $op --sizes $S \
        --iters 20 --warmup 5 --algorithms auto $( [ $LL = 262144 ] && echo --nccl ) 2>/dev/null | grep -E "^$op" | sed "s/^/ll$LL,/"
    done
  done > gpurun_out/l4_p$N.csv
done
cat gpurun_out/l4_p4.csv gpurun_out/l4_p2.csv
