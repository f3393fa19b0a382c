# device-count gathers: p = 4 / 2 processes, p = 1, co-located p = 8
cd $GRAFT_REPO_ROOT
timeout 500 python tests/gpu_launch.py 4 gathers,all_to_allv,baseline > gpurun_out/g1_p4.log 2>&1; echo p4 rc=$?; tail -4 gpurun_out/g1_p4.log
CUDA_VISIBLE_DEVICES=0,1 timeout 300 python tests/gpu_launch.py 2 gathers > gpurun_out/g1_p2.log 2>&1; echo p2 rc=$?; tail -2 gpurun_out/g1_p2.log
timeout 300 python tests/gpu_launch.py 1 gathers > gpurun_out/g1_p1.log 2>&1; echo p1 rc=$?; tail -1 gpurun_out/g1_p1.log
CUDA_VISIBLE_DEVICES=0 MCRDL_LAUNCH_TIMEOUT=500 timeout 560 python tests/gpu_launch.py 8 gathers --colocated > gpurun_out/g1_co8.log 2>&1; echo co8 rc=$?; tail -2 gpurun_out/g1_co8.log
grep -h "FAIL\|mismatch\|Error" gpurun_out/g1_*.log | head -20
