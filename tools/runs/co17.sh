cd $GRAFT_REPO_ROOT
free -g | head -2; nproc
export MCRDL_LAUNCH_TIMEOUT=400 MCRDL_DEBUG=1
( time MCRDL_COLOCATED_LOG=gpurun_out/co17_p2p4.log timeout 430 python tests/gpu_launch.py 4 p2p --colocated ) > gpurun_out/co17_4.log 2>&1
echo "== p2p 4"; grep -h "rank .: exit\|^real" gpurun_out/co17_4.log
grep -h "mcrdl\]" gpurun_out/co17_p2p4.log | grep -v "comm 0x" | sort | uniq -c | sort -rn | head -12
grep -A6 "^    [a-z]" gpurun_out/co17_4.log | grep -v "^  File\|^   *\^" | head -20
for w in 2 8; do
( time MCRDL_COLOCATED_LOG=gpurun_out/co17_b$w.log timeout 430 python tests/gpu_launch.py $w baseline,large --colocated ) > gpurun_out/co17_b_$w.log 2>&1
echo "== baseline,large $w"; grep -h "rank .: exit\|^real" gpurun_out/co17_b_$w.log
grep -A6 "^    [a-z]" gpurun_out/co17_b_$w.log | grep -v "^  File\|^   *\^" | head -20
done
