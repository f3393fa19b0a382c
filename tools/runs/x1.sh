# exchange A/B: per-peer (eager) flags vs per-row flags, p = 4 and 2; parity
cd $GRAFT_REPO_ROOT
for N in 4 2; do
for E in 1 0; do
MCRDL_X_EAGER=$E CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops all_to_allv,all_gatherv --sizes 1M,4M,16M,64M,256M,1G --iters 20 --warmup 5 --algorithms auto 2>/dev/null | grep -E "^all_" | sed "s/^/eager$E,/"
done
done > gpurun_out/x1.csv; cat gpurun_out/x1.csv
timeout 500 python tests/gpu_launch.py 4 all_to_allv,all_to_all,baseline,codec,gathers,bcast_scatter,a3 > gpurun_out/x1_par4.log 2>&1; echo par4 rc=$?; tail -3 gpurun_out/x1_par4.log
timeout 400 python tests/gpu_launch.py 2 all_to_allv,all_to_all,codec,gathers > gpurun_out/x1_par2.log 2>&1; echo par2 rc=$?; tail -3 gpurun_out/x1_par2.log
