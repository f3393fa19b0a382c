cd $GRAFT_REPO_ROOT
( time timeout 1700 python -m pytest tests -m gpu -q --durations=0 ) > gpurun_out/t2_pytest.log 2>&1
tail -25 gpurun_out/t2_pytest.log
