# chain bcast at p = 2 vs direct write
cd $GRAFT_REPO_ROOT
CUDA_VISIBLE_DEVICES=0,1 timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops bcast --sizes 1M,4M,16M,64M,256M,1G --iters 10 --warmup 3 --algorithms chain,direct_write --nccl 2>/dev/null | grep -E "^bcast" > gpurun_out/g4.csv; cat gpurun_out/g4.csv
CUDA_VISIBLE_DEVICES=0,1 timeout 300 python tests/gpu_launch.py 2 bcast_scatter > gpurun_out/g4_par2.log 2>&1; echo par2 rc=$?; head -2 gpurun_out/g4_par2.log
