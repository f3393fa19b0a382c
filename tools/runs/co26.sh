cd $GRAFT_REPO_ROOT
export MCRDL_LAUNCH_TIMEOUT=150 MCRDL_TIMEOUT_SECS=5
for parts in ring,queued,rendezvous,pingpong,self,host graph,lenm ring,queued,rendezvous ring,graph; do
( MCRDL_P2P_PARTS=$parts timeout 170 python tests/gpu_launch.py 2 p2p,symm --colocated ) > gpurun_out/co26.log 2>&1
echo "== $parts"; grep -h "rank .: exit" gpurun_out/co26.log
done
