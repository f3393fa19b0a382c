# chain bcast parity at p = 2 (processes and co-located), then the 1-GPU-box suite
cd $GRAFT_REPO_ROOT
CUDA_VISIBLE_DEVICES=0,1 timeout 300 python tests/gpu_launch.py 2 bcast_scatter > gpurun_out/g5_par2.log 2>&1; echo par2 rc=$?; head -2 gpurun_out/g5_par2.log
CUDA_VISIBLE_DEVICES=0 MCRDL_LAUNCH_TIMEOUT=250 timeout 300 python tests/gpu_launch.py 2 bcast_scatter --colocated > gpurun_out/g5_co2.log 2>&1; echo co2 rc=$?; head -2 gpurun_out/g5_co2.log
CUDA_VISIBLE_DEVICES=0 bash -c '( time timeout 1500 python -m pytest tests -m gpu -q --durations=0 ) > gpurun_out/g5_pytest_1gpu.log 2>&1'; grep -E "passed|failed" gpurun_out/g5_pytest_1gpu.log | tail -2
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g5_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/g5_smoke.log
