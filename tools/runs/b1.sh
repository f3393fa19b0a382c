cd $GRAFT_REPO_ROOT
run() { timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops all_reduce --iters 10 --warmup 3 "$@" 2>/dev/null | grep -E "^all_reduce"; }
echo "== default"; run --sizes 16M,64M,256M,1G --algorithms two_shot,nvls
echo "== nvls 4GiB buffer"; MCRDL_NVLS_BYTES=4294967296 run --sizes 256M,1G --algorithms nvls
echo "== chunk 256"; MCRDL_AR_CHUNK_KB=256 run --sizes 16M,64M --algorithms two_shot
echo "== chunk 64"; MCRDL_AR_CHUNK_KB=64 run --sizes 16M,64M --algorithms two_shot
echo "== nvls gp 48"; MCRDL_NVLS_GP=48 run --sizes 64M,256M,1G --algorithms nvls
echo "== nvls gp 24"; MCRDL_NVLS_GP=24 run --sizes 64M,256M,1G --algorithms nvls
