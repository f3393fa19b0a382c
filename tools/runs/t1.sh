cd $GRAFT_REPO_ROOT
( time timeout 1700 python -m pytest tests -m gpu -x -q --durations=0 ) > gpurun_out/t1_pytest.log 2>&1
tail -30 gpurun_out/t1_pytest.log
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/t1_smoke.log 2>&1; tail -5 gpurun_out/t1_smoke.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/t1_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t1_ncu_smoke.log 2>&1; echo ncu_rc=$?; tail -3 gpurun_out/t1_ncu_smoke.log
grep -o '"mcrdl::[a-z_]*' gpurun_out/t1_launches.csv | sort | uniq -c
