# Final verification at HEAD (4xB200): GPU suite, smoke, bench N=1/2/4, bcast + all_reduce sweep at p = 4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -m gpu -q --durations=0 ) > gpurun_out/v4_pytest.log 2>&1
grep -E "passed|failed" gpurun_out/v4_pytest.log | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v4_smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/v4_bench_n1.log 2>&1; echo bench1 rc=$?
for N in 2 4; do
CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29504 bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/v4_bench_n$N.log 2>&1; echo "bench n$N rc=$?"
done
python - <<'PY'
import json
for f in ['v4_bench_n1','v4_bench_n2','v4_bench_n4']:
    try:
        l=[x for x in open('gpurun_out/'+f+'.log') if x.startswith('{')][-1]; d=json.loads(l)
        print(f, 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'frac', d.get('roofline',{}).get('frac'), 'launches', d.get('gpu_launches'))
    except Exception as e:
        print(f, 'ERR', e)
PY
for op in bcast all_reduce; do
timeout 400 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29575 -m paper_2303_08374_b200.tuner --ops $op --sizes 8,4K,256K,1M,2M,4M,16M,64M,256M,1G --iters 10 --warmup 3 --algorithms auto --nccl 2>/dev/null | grep -E "^$op"
done > gpurun_out/v4_sweep_p4.csv; cat gpurun_out/v4_sweep_p4.csv
