cd $GRAFT_REPO_ROOT
export MCRDL_LAUNCH_TIMEOUT=300
( time MCRDL_COLOCATED_LOG=gpurun_out/co18_p2p4.log timeout 330 python tests/gpu_launch.py 4 p2p --colocated ) > gpurun_out/co18_4.log 2>&1
echo "== p2p 4"; grep -h "rank .: exit\|^real" gpurun_out/co18_4.log
grep -h "mcrdl\]" gpurun_out/co18_p2p4.log | grep -v "comm 0x" | sort | uniq -c | sort -rn | head -6
( time MCRDL_MAX_SMS=8 MCRDL_COLOCATED_LOG=gpurun_out/co18_p2p4b.log timeout 330 python tests/gpu_launch.py 4 p2p --colocated ) > gpurun_out/co18_4b.log 2>&1
echo "== p2p 4 maxsms 8"; grep -h "rank .: exit\|^real" gpurun_out/co18_4b.log
grep -h "mcrdl\]" gpurun_out/co18_p2p4b.log | grep -v "comm 0x" | sort | uniq -c | sort -rn | head -6
( time MCRDL_COLOCATED_LOG=gpurun_out/co18_b2.log timeout 330 python tests/gpu_launch.py 2 baseline --colocated ) > gpurun_out/co18_b_2.log 2>&1
echo "== baseline 2"; grep -h "rank .: exit\|^real" gpurun_out/co18_b_2.log; tail -5 gpurun_out/co18_b2.log
