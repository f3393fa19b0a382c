set -x
cd $GRAFT_REPO_ROOT
nvidia-smi -L
( time timeout 300 python tests/gpu_launch.py 2 smoke --colocated ) > gpurun_out/co_smoke2.log 2>&1
( time timeout 900 python tests/gpu_launch.py 2 --colocated ) > gpurun_out/co_all2.log 2>&1
( time timeout 900 python tests/gpu_launch.py 8 --colocated ) > gpurun_out/co_all8.log 2>&1
ncu --metrics gpu__time_duration.sum -c 5 python -c "import os; print({k:v for k,v in os.environ.items() if 'INJ' in k or 'NV_' in k or 'NSIGHT' in k})" > gpurun_out/ncu_env.log 2>&1
tail -3 gpurun_out/co_*.log
