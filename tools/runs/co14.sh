cd $GRAFT_REPO_ROOT
export MCRDL_LAUNCH_TIMEOUT=150
for sc in async_fusion,graphs host_buffers,graphs reduce_family,graphs golden,all_reduce,all_to_allv,all_to_all,gathers,bcast_scatter,graphs; do
( time timeout 170 python tests/gpu_launch.py 4 $sc --colocated ) > gpurun_out/co14.log 2>&1
echo "== $sc"; grep -h "rank .: exit\|^real" gpurun_out/co14.log
done
