# chain bcast geometry A/B (p = 4): CTAs x chunk KiB
cd $GRAFT_REPO_ROOT
N=4
for CFG in "128 256" "128 64" "128 128" "256 64" "256 128" "64 64"; do
set -- $CFG
MCRDL_BCAST_CHAIN_CTAS=$1 MCRDL_BCAST_CHAIN_KB=$2 timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops bcast --sizes 4M,16M,64M,256M,1G --iters 10 --warmup 3 --algorithms chain 2>/dev/null | grep -E "^bcast" | sed "s/^/c$1k$2,/"
done > gpurun_out/g3_chain.csv; cat gpurun_out/g3_chain.csv
