cd $GRAFT_REPO_ROOT
export MCRDL_DEBUG=1
( time MCRDL_COLOCATED_LOG=gpurun_out/co7_full2.log timeout 300 python tests/gpu_launch.py 2 reduce_family --colocated ) > gpurun_out/co7_2.log 2>&1
( time MCRDL_COLOCATED_LOG=gpurun_out/co7_full8.log timeout 400 python tests/gpu_launch.py 8 golden,all_reduce --colocated ) > gpurun_out/co7_8.log 2>&1
grep -h "rank .: exit\|^real" gpurun_out/co7_*.log
grep -h "mcrdl\]" gpurun_out/co7_full*.log | grep -v "comm 0x" | head -30
