cd $GRAFT_REPO_ROOT
export MCRDL_WORKER_DUMP_SECS=60 MCRDL_LAUNCH_TIMEOUT=300
for w in 4 8 2; do
( time MCRDL_COLOCATED_LOG=gpurun_out/co12_full$w.log timeout 330 python tests/gpu_launch.py $w --colocated ) > gpurun_out/co12_$w.log 2>&1
grep -h "rank .: exit\|^real" gpurun_out/co12_$w.log
grep -h "mcrdl\]" gpurun_out/co12_full$w.log | grep -v "comm 0x" | head -5
grep -A3 "^    [a-z]" gpurun_out/co12_$w.log | head -40
done
