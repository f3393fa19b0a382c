cd $GRAFT_REPO_ROOT
timeout 300 python tests/gpu_launch.py 4 commlog,all_to_allv,golden > gpurun_out/l3_parity.log 2>&1; echo parity rc=$?; head -4 gpurun_out/l3_parity.log
S=8,4K,32K,256K,1M
for N in 4 2; do
  DEV=$(seq -s, 0 $((N-1)))
  for op in all_reduce all_to_allv bcast; do
    CUDA_VISIBLE_DEVICES=$DEV timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops $op --sizes $S \
      --iters 20 --warmup 5 --algorithms auto --nccl 2>/dev/null | grep -E "^$op"
  done > gpurun_out/l3_lat_p$N.csv
done
cat gpurun_out/l3_lat_p4.csv gpurun_out/l3_lat_p2.csv
