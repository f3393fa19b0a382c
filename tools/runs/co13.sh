cd $GRAFT_REPO_ROOT
export MCRDL_LAUNCH_TIMEOUT=200 MCRDL_DEBUG=1
( time MCRDL_COLOCATED_LOG=gpurun_out/co13_full4.log timeout 230 python tests/gpu_launch.py 4 --colocated ) > gpurun_out/co13_4.log 2>&1
grep -h "rank .: exit\|^real" gpurun_out/co13_4.log
grep -h "mcrdl\]" gpurun_out/co13_full4.log | grep -v "LL timeout\|flag timeout" | head -30
grep -h "mcrdl\]" gpurun_out/co13_full4.log | grep "timeout" | awk '{print $1,$2,$3,$4,$5,$9,$10}' | sort | uniq -c | head
grep -B2 -A12 "^    graph" gpurun_out/co13_4.log | grep -v "^  File\|^   *\^" | head -60
