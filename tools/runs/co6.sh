cd $GRAFT_REPO_ROOT
export MCRDL_DEBUG=1
( time timeout 900 python tests/gpu_launch.py 2 --colocated ) > gpurun_out/co6_all2.log 2>&1
( time timeout 900 python tests/gpu_launch.py 4 --colocated ) > gpurun_out/co6_all4.log 2>&1
( time timeout 900 python tests/gpu_launch.py 8 --colocated ) > gpurun_out/co6_all8.log 2>&1
grep -h "rank .: exit\|^real" gpurun_out/co6_*.log
