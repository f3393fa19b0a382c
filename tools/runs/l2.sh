cd $GRAFT_REPO_ROOT
S=8,4K,32K,256K,1M
for cfg in "2 1" "1 1" "1 0" "2 0" "4 1"; do
  set -- $cfg
  for op in all_to_allv bcast all_reduce; do
    MCRDL_LL_X_UPT=$1 MCRDL_LOG=$2 timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 \
      --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops $op --sizes $S \
      --iters 20 --warmup 5 --algorithms auto 2>/dev/null | grep -E "^$op" | sed "s/^/upt$1,log$2,/"
  done
done > gpurun_out/l2.csv
cat gpurun_out/l2.csv
