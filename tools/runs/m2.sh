cd $GRAFT_REPO_ROOT
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum"
for w in 2 4; do
  timeout 600 python tools/ncu_multi.py --world $w --out gpurun_out/m2_ncu_p$w --metrics "$M" > gpurun_out/m2_ncu_p$w.log 2>&1
  echo "ncu p$w rc=$?"; tail -2 gpurun_out/m2_ncu_p$w.log; grep -c . gpurun_out/m2_ncu_p$w.csv
done
# N = 1: k_copy at the current geometry, full set (traffic for roofline)
timeout 600 ncu --set full --clock-control none -k regex:k_copy -c 1 --csv --page raw --log-file gpurun_out/m2_kcopy_raw.csv python bench.py --gpus 1 --steps 2 --warmup 1 > gpurun_out/m2_kcopy.log 2>&1; echo kcopy_rc=$?
# sanitizers on the p = 2 smoke (one process per GPU)
for tool in memcheck racecheck synccheck; do
  MCRDL_TIMEOUT_SECS=120 timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python tests/gpu_launch.py 2 smoke > gpurun_out/m2_san_$tool.log 2>&1; echo "$tool rc=$?"; tail -4 gpurun_out/m2_san_$tool.log
done
( time timeout 1500 python -m pytest tests -m gpu -q --durations=0 ) > gpurun_out/m2_pytest.log 2>&1
tail -22 gpurun_out/m2_pytest.log
S=8,4K,32K,256K,1M,16M,64M,256M,1G
for N in 4 2; do
  DEV=$(seq -s, 0 $((N-1)))
  for op in all_reduce all_to_allv bcast; do
    CUDA_VISIBLE_DEVICES=$DEV timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops $op --sizes $S \
      --iters 10 --warmup 3 --nccl 2>/dev/null | grep -E "^$op"
  done > gpurun_out/m2_sweep_p$N.csv
  wc -l gpurun_out/m2_sweep_p$N.csv
done
