cd $GRAFT_REPO_ROOT
S=8,4K,32K,256K
for LOG in 1 0; do
  for op in all_reduce all_to_allv bcast; do
    MCRDL_LOG=$LOG timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 \
      --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops $op --sizes $S \
      --iters 20 --warmup 5 --algorithms auto 2>/dev/null | grep -E "^$op"
  done > gpurun_out/l1_log$LOG.csv
done
paste -d' ' gpurun_out/l1_log1.csv gpurun_out/l1_log0.csv
