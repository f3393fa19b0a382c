cd $GRAFT_REPO_ROOT
for w in 2 4 8; do
( time MCRDL_COLOCATED_LOG=gpurun_out/co8_full$w.log timeout 600 python tests/gpu_launch.py $w --colocated ) > gpurun_out/co8_$w.log 2>&1
done
grep -h "rank .: exit\|^real" gpurun_out/co8_?.log
grep -h "mcrdl\]" gpurun_out/co8_full*.log | grep -v "comm 0x" | head -20
