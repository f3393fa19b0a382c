cd $GRAFT_REPO_ROOT
export MCRDL_TIMEOUT_SECS=5 MCRDL_MASTER_PORT=29611
timeout 120 python tools/runs/co_debug.py 2 1048576,4194304,8388608,16777216,25165829 two_shot > gpurun_out/dbg_a.log 2>&1
export MCRDL_MASTER_PORT=29612
CUDA_MODULE_LOADING=EAGER timeout 120 python tools/runs/co_debug.py 2 1048576,4194304,8388608,16777216,25165829 two_shot > gpurun_out/dbg_b.log 2>&1
export MCRDL_MASTER_PORT=29613
MCRDL_MAX_SMS=20 timeout 120 python tools/runs/co_debug.py 2 1048576,4194304,8388608,16777216,25165829 two_shot > gpurun_out/dbg_c.log 2>&1
export MCRDL_MASTER_PORT=29614
timeout 120 python tools/runs/co_debug.py 8 1,1000,65536,1048576 auto > gpurun_out/dbg_d.log 2>&1
export MCRDL_MASTER_PORT=29615
timeout 120 python tools/runs/co_debug.py 8 1000,1048576,4194304 one_shot > gpurun_out/dbg_e.log 2>&1
export MCRDL_MASTER_PORT=29616
timeout 120 python tools/runs/co_debug.py 8 1048576,4194304 two_shot > gpurun_out/dbg_f.log 2>&1
cuobjdump --dump-resource-usage paper_2303_08374_b200/lib/libmcrdl_nvl.so 2>&1 | grep -A1 "k_ar_pipe\|k_exchange\|k_ar_ll\|k_ar_oneshot" | grep -o "REG:[0-9]*\|SHARED:[0-9]*\|Function [^:]*" | paste - - - | sort | uniq | head -40 > gpurun_out/resusage.log
tail -n 30 gpurun_out/dbg_*.log
