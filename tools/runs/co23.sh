cd $GRAFT_REPO_ROOT
export MCRDL_LAUNCH_TIMEOUT=300
( time MCRDL_COLOCATED_LOG=gpurun_out/co23_full.log timeout 330 python tests/gpu_launch.py 2 all_reduce,symm --colocated ) > gpurun_out/co23.log 2>&1
grep -h "rank .: exit\|^real\|     log" gpurun_out/co23.log | tail -90
