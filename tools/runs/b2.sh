cd $GRAFT_REPO_ROOT
run() { N=$1; shift; CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --iters 10 --warmup 3 "$@" 2>/dev/null | grep -E "^(all_reduce|all_to_allv)"; }
echo "== p2 default ws"; run 2 --ops all_reduce --sizes 256M,1G --algorithms two_shot
echo "== p2 ws 4G"; MCRDL_NVL_WORKSPACE_BYTES=4294967296 run 2 --ops all_reduce --sizes 256M,1G --algorithms two_shot
echo "== p4 ws 4G two_shot"; MCRDL_NVL_WORKSPACE_BYTES=4294967296 run 4 --ops all_reduce --sizes 1G --algorithms two_shot
echo "== p4 a2av default"; run 4 --ops all_to_allv --sizes 256M,1G
echo "== p4 a2av ws 4G"; MCRDL_NVL_WORKSPACE_BYTES=4294967296 run 4 --ops all_to_allv --sizes 256M,1G
echo "== p4 nvls 4G bf16"; MCRDL_NVLS_BYTES=4294967296 run 4 --ops all_reduce --sizes 64M,1G --algorithms nvls --dtype bf16
