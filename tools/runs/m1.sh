cd $GRAFT_REPO_ROOT
nvidia-smi -L
ncu --query-metrics --chip gb100 > gpurun_out/m1_metrics.txt 2>&1 || ncu --query-metrics > gpurun_out/m1_metrics.txt 2>&1
grep -i "^nvl\|nvlink" gpurun_out/m1_metrics.txt | head -20
NVL=$(grep -oE "^nvl[a-z]*__[a-z_]*bytes[a-z_]*" gpurun_out/m1_metrics.txt | sort -u | head -4 | sed 's/$/.sum/' | paste -sd, -)
echo "NVL metrics: $NVL"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
[ -n "$NVL" ] && M="$M,$NVL"
for w in 2 4; do
  timeout 600 python tools/ncu_multi.py --world $w --out gpurun_out/m1_ncu_p$w --metrics "$M" > gpurun_out/m1_ncu_p$w.log 2>&1 || \
  timeout 600 python tools/ncu_multi.py --world $w --out gpurun_out/m1_ncu_p$w --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum > gpurun_out/m1_ncu_p${w}b.log 2>&1
  tail -3 gpurun_out/m1_ncu_p$w.log
done
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29$((500+n)) bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/m1_bench_n$n.log 2>&1; echo "bench n=$n rc=$?"
  tail -c 600 gpurun_out/m1_bench_n$n.log
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29$((600+n)) bench.py --impl reference --gpus $n --steps 20 --warmup 5 > gpurun_out/m1_ref_n$n.log 2>&1; echo "ref n=$n rc=$?"
  tail -c 400 gpurun_out/m1_ref_n$n.log
done
( time timeout 1500 python -m pytest tests -m gpu -q --durations=0 ) > gpurun_out/m1_pytest.log 2>&1
tail -25 gpurun_out/m1_pytest.log
