cd $GRAFT_REPO_ROOT
export MCRDL_LAUNCH_TIMEOUT=200
for sc in p2p,symm graphs,symm host_buffers,async_fusion,symm golden,all_reduce,all_to_allv,all_to_all,gathers,bcast_scatter,reduce_family,symm; do
( time timeout 230 python tests/gpu_launch.py 2 $sc --colocated ) > gpurun_out/co24.log 2>&1
echo "== $sc"; grep -h "rank .: exit\|^real" gpurun_out/co24.log
done
