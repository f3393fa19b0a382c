cd $GRAFT_REPO_ROOT
export MCRDL_DEBUG=1
( time timeout 900 python tests/gpu_launch.py 2 golden,all_reduce,all_to_allv,all_to_all,gathers --colocated ) > gpurun_out/co4_a2.log 2>&1
grep -h "rank .: exit\|^real" gpurun_out/co4_*.log
grep -h "mcrdl\]" gpurun_out/co4_a2.log | head -50
