cd $GRAFT_REPO_ROOT
export MCRDL_WORKER_DUMP_SECS=45 MCRDL_LAUNCH_TIMEOUT=200
( time MCRDL_COLOCATED_LOG=gpurun_out/co10_full2.log timeout 260 python tests/gpu_launch.py 2 --colocated ) > gpurun_out/co10_2.log 2>&1
grep -h "rank .: exit\|^real" gpurun_out/co10_2.log
grep -h "mcrdl\]" gpurun_out/co10_full2.log | grep -v "comm 0x" | head -10
grep -A3 "^    [a-z]" gpurun_out/co10_2.log | head -80
