cd $GRAFT_REPO_ROOT
export MCRDL_LAUNCH_TIMEOUT=400
for i in 1 2 3; do
( time MCRDL_COLOCATED_LOG=gpurun_out/co22_full$i.log timeout 430 python tests/gpu_launch.py 2 --colocated ) > gpurun_out/co22_$i.log 2>&1
echo "== run $i"; grep -h "rank .: exit\|^real" gpurun_out/co22_$i.log
grep -h "timeout:" gpurun_out/co22_full$i.log | awk '{print $2, $3, $4, $5, $9, $10}' | sort | uniq -c | sort -rn | head -4
grep -E "^    [a-z]" gpurun_out/co22_$i.log | grep -v "File\|return\|self\.\|chk\|raise\|cx\.\|SCEN\|inst\.\|_lib" | sort | uniq -c | head
done
