# one-shot geometry A/B: CTA cap x packs per thread, p = 4 and 2
cd $GRAFT_REPO_ROOT
for N in 4 2; do
for CFG in "64 2" "128 1" "148 1" "296 1" "128 2" "296 2"; do
set -- $CFG
MCRDL_AR_ONESHOT_CTAS=$1 MCRDL_AR_ONESHOT_PPT=$2 CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops all_reduce --sizes 256K,512K,1M,2M,4M,8M --iters 30 --warmup 5 --algorithms one_shot 2>/dev/null | grep -E "^all_" | sed "s/^/c$1p$2,/"
done
CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops all_reduce --sizes 256K,512K,1M,2M,4M,8M --iters 30 --warmup 5 --algorithms two_shot --nccl 2>/dev/null | grep -E "^all_" | sed "s/^/ref,/"
done > gpurun_out/o1.csv; cat gpurun_out/o1.csv
