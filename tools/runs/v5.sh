cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "all_scenarios or tma_senders" > gpurun_out/v5_pytest_procs.log 2>&1; grep -E "passed|failed" gpurun_out/v5_pytest_procs.log | tail -2
