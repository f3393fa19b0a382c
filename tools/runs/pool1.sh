cd $GRAFT_REPO_ROOT
timeout 300 python tests/gpu_launch.py 4 pool,symm > gpurun_out/pool_p4.log 2>&1; echo p4 rc=$?; head -6 gpurun_out/pool_p4.log
MCRDL_LAUNCH_TIMEOUT=250 timeout 300 python tests/gpu_launch.py 2 pool --colocated > gpurun_out/pool_co2.log 2>&1; echo co2 rc=$?; head -4 gpurun_out/pool_co2.log
