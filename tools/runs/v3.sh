# Round-end verification at HEAD on a 4xB200 box: GPU suite, bench N=1/2/4,
# reference arm N=4, then the per-op sweep with NCCL (tools/final_sweep.sh).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests -m gpu -q --durations=0 ) > gpurun_out/v3_pytest.log 2>&1
tail -4 gpurun_out/v3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v3_smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/v3_bench_n1.log 2>&1; echo bench1 rc=$?
for N in 2 4; do
CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29504 bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/v3_bench_n$N.log 2>&1; echo "bench n$N rc=$?"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29505 bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > gpurun_out/v3_ref_n4.log 2>&1; echo "ref n4 rc=$?"
python - <<'PY'
import json
for f in ['v3_bench_n1','v3_bench_n2','v3_bench_n4','v3_ref_n4']:
    try:
        l=[x for x in open('gpurun_out/'+f+'.log') if x.startswith('{')][-1]; d=json.loads(l)
        print(f, 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'frac', d.get('roofline',{}).get('frac'), 'cpu', (d.get('cpu_baseline') or {}).get('value'))
    except Exception as e:
        print(f, 'ERR', e)
PY
bash tools/final_sweep.sh
