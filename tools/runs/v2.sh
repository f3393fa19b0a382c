cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -m gpu -q --durations=0 ) > gpurun_out/v2_pytest.log 2>&1
tail -18 gpurun_out/v2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v2_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/v2_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/v2_bench_n1.log 2>&1; echo bench rc=$?; tail -c 1500 gpurun_out/v2_bench_n1.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/v2_ref_n1.log 2>&1; echo ref rc=$?; tail -c 600 gpurun_out/v2_ref_n1.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v2_launches_n1.csv python bench.py --steps 3 --warmup 3 > gpurun_out/v2_ncu_launch.log 2>&1; echo ncu-launch rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_copy --launch-skip 4 -c 1 -o gpurun_out/v2_kcopy -f python bench.py --steps 3 --warmup 3 > gpurun_out/v2_ncu_full.log 2>&1; echo ncu-full rc=$?
