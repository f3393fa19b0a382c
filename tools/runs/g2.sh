# device-count gathers (p = 4 / 2 processes, p = 1, co-located p = 8) + chain bcast parity and A/B
cd $GRAFT_REPO_ROOT
timeout 500 python tests/gpu_launch.py 4 gathers,bcast_scatter > gpurun_out/g2_p4.log 2>&1; echo p4 rc=$?; head -4 gpurun_out/g2_p4.log
CUDA_VISIBLE_DEVICES=0,1 timeout 300 python tests/gpu_launch.py 2 gathers > gpurun_out/g2_p2.log 2>&1; echo p2 rc=$?; head -2 gpurun_out/g2_p2.log
timeout 300 python tests/gpu_launch.py 1 gathers > gpurun_out/g2_p1.log 2>&1; echo p1 rc=$?; head -1 gpurun_out/g2_p1.log
CUDA_VISIBLE_DEVICES=0 MCRDL_LAUNCH_TIMEOUT=500 timeout 560 python tests/gpu_launch.py 8 gathers,bcast_scatter --colocated > gpurun_out/g2_co8.log 2>&1; echo co8 rc=$?; head -2 gpurun_out/g2_co8.log
grep -h "Error\|FAIL" gpurun_out/g2_*.log | head -10
for N in 4 3; do
for CFG in "64 256" "32 256" "128 256" "64 1024"; do
set -- $CFG
MCRDL_BCAST_CHAIN_CTAS=$1 MCRDL_BCAST_CHAIN_KB=$2 CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops bcast --sizes 1M,4M,16M,64M,256M,1G --iters 10 --warmup 3 --algorithms chain 2>/dev/null | grep -E "^bcast" | sed "s/^/c$1k$2,/"
done
CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops bcast --sizes 1M,4M,16M,64M,256M,1G --iters 10 --warmup 3 --algorithms direct_write,nvls --nccl 2>/dev/null | grep -E "^bcast" | sed "s/^/ref,/"
done > gpurun_out/g2_chain.csv; cat gpurun_out/g2_chain.csv
