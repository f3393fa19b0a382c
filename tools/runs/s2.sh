cd $GRAFT_REPO_ROOT
for N in 4 2; do
CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops all_to_allv --sizes 16M,64M,256M,1G --iters 10 --warmup 3 --algorithms auto 2>/dev/null | grep -E "^all_to_allv"
CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops all_reduce --sizes 256M,1G --iters 10 --warmup 3 --algorithms two_shot 2>/dev/null | grep -E "^all_reduce"
done > gpurun_out/s2.csv; cat gpurun_out/s2.csv
timeout 400 python tests/gpu_launch.py 4 all_to_allv,large,all_to_all > gpurun_out/s2_par4.log 2>&1; echo par4 rc=$?; head -2 gpurun_out/s2_par4.log
timeout 400 python tests/gpu_launch.py 2 large,gathers > gpurun_out/s2_par2.log 2>&1; echo par2 rc=$?; head -2 gpurun_out/s2_par2.log
