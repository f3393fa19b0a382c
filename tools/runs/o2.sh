# one-shot with batched loads: geometry A/B, p = 4 and 2; parity
cd $GRAFT_REPO_ROOT
for N in 4 2; do
for CFG in "64 2" "128 1" "128 2" "148 1"; do
set -- $CFG
MCRDL_AR_ONESHOT_CTAS=$1 MCRDL_AR_ONESHOT_PPT=$2 CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops all_reduce --sizes 128K,256K,512K,1M,2M,4M,8M --iters 30 --warmup 5 --algorithms one_shot 2>/dev/null | grep -E "^all_" | sed "s/^/c$1p$2,/"
done
CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops all_reduce --sizes 128K,256K,512K,1M,2M,4M,8M --iters 30 --warmup 5 --algorithms two_shot --nccl 2>/dev/null | grep -E "^all_" | sed "s/^/ref,/"
done > gpurun_out/o2.csv; cat gpurun_out/o2.csv
timeout 500 python tests/gpu_launch.py 4 all_reduce,async_fusion,baseline > gpurun_out/o2_par4.log 2>&1; echo par4 rc=$?; tail -3 gpurun_out/o2_par4.log
MCRDL_AR_ONESHOT_CTAS=128 MCRDL_AR_ONESHOT_PPT=1 timeout 400 python tests/gpu_launch.py 2 all_reduce,async_fusion > gpurun_out/o2_par2.log 2>&1; echo par2 rc=$?; tail -3 gpurun_out/o2_par2.log
