cd $GRAFT_REPO_ROOT
( time timeout 1500 python -m pytest tests -m gpu -q --durations=0 ) > gpurun_out/f1_pytest.log 2>&1
tail -20 gpurun_out/f1_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/f1_bench_n1.log 2>&1; echo "bench n1 rc=$?"
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29$((500+n)) bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/f1_bench_n$n.log 2>&1; echo "bench n$n rc=$?"
done
S=8,4K,32K,128K,256K,1M,16M,64M,256M,1G
for N in 4 2; do
  DEV=$(seq -s, 0 $((N-1)))
  for op in all_reduce all_to_allv all_gatherv bcast; do
    CUDA_VISIBLE_DEVICES=$DEV timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops $op --sizes $S \
      --iters 10 --warmup 3 --algorithms auto --nccl 2>/dev/null | grep -E "^$op"
  done > gpurun_out/f1_sweep_p$N.csv
  wc -l gpurun_out/f1_sweep_p$N.csv
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f1_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f1_ncu_smoke.log 2>&1; echo ncu_rc=$?
