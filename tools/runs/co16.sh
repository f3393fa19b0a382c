cd $GRAFT_REPO_ROOT
export MCRDL_LAUNCH_TIMEOUT=200 MCRDL_DEBUG=1
( time MCRDL_COLOCATED_LOG=gpurun_out/co16_full4.log timeout 230 python tests/gpu_launch.py 4 p2p --colocated ) > gpurun_out/co16_4.log 2>&1
grep -h "rank .: exit\|^real" gpurun_out/co16_4.log
grep -h "mcrdl\]" gpurun_out/co16_full4.log | sort | uniq -c | sort -rn | head -30
grep -A8 "^    [a-z]" gpurun_out/co16_4.log | grep -v "^  File\|^   *\^" | head -30
