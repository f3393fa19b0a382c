cd $GRAFT_REPO_ROOT
for SM in 148 74 48 32; do
  MCRDL_MAX_SMS=$SM timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops all_to_allv --sizes 16M,64M,256M,1G --iters 10 --warmup 3 --algorithms auto 2>/dev/null | grep -E "^all_to_allv" | sed "s/^/sms$SM,/"
  MCRDL_MAX_SMS=$SM timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops all_reduce --sizes 64M,256M --iters 10 --warmup 3 --algorithms two_shot,nvls 2>/dev/null | grep -E "^all_reduce" | sed "s/^/sms$SM,/"
done > gpurun_out/s1.csv
cat gpurun_out/s1.csv
