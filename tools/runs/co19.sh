cd $GRAFT_REPO_ROOT
export MCRDL_LAUNCH_TIMEOUT=400
for w in 4 8 2; do
( time MCRDL_COLOCATED_LOG=gpurun_out/co19_full$w.log timeout 430 python tests/gpu_launch.py $w --colocated ) > gpurun_out/co19_$w.log 2>&1
echo "== $w"; grep -h "rank .: exit\|^real" gpurun_out/co19_$w.log
grep -h "mcrdl\]" gpurun_out/co19_full$w.log | grep -v "comm 0x" | sort | uniq -c | sort -rn | head -6
grep -A6 "^    [a-z]" gpurun_out/co19_$w.log | grep -v "^  File\|^   *\^" | head -24
done
