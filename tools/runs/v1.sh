cd $GRAFT_REPO_ROOT
( time timeout 1500 python -m pytest tests -m gpu -q --durations=0 ) > gpurun_out/v1_pytest.log 2>&1
tail -18 gpurun_out/v1_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/v1_bench_n1.log 2>&1; echo bench rc=$?; tail -c 1500 gpurun_out/v1_bench_n1.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/v1_ref_n1.log 2>&1; echo ref rc=$?; tail -c 600 gpurun_out/v1_ref_n1.log
