cd $GRAFT_REPO_ROOT
export MCRDL_LAUNCH_TIMEOUT=200
( time MCRDL_COLOCATED_LOG=gpurun_out/co25_full.log timeout 230 python tests/gpu_launch.py 2 p2p,symm --colocated ) > gpurun_out/co25.log 2>&1
grep -h "rank .: exit\|^real" gpurun_out/co25.log
grep -E "^    [a-z]" gpurun_out/co25.log | grep -v "File\|return\|self\.\|chk\|raise\|cx\.\|SCEN\|inst\.\|_lib" | head
grep "     log" gpurun_out/co25.log | tail -30
grep "timeout:" gpurun_out/co25_full.log | awk '{print $1,$2,$3,$4,$5,$9,$10}' | sort | uniq -c | head
