cd $GRAFT_REPO_ROOT
( time timeout 900 python tests/gpu_launch.py 2 --colocated ) > gpurun_out/co3_all2.log 2>&1
( time CUDA_MODULE_LOADING=EAGER timeout 900 python tests/gpu_launch.py 2 --colocated ) > gpurun_out/co3_all2_eager.log 2>&1
( time timeout 900 python tests/gpu_launch.py 8 --colocated ) > gpurun_out/co3_all8.log 2>&1
grep -h "rank .: exit\|^real" gpurun_out/co3_*.log
