cd $GRAFT_REPO_ROOT
export MCRDL_DEBUG=1 MCRDL_TIMEOUT_SECS=10 CUDA_MODULE_DATA_LOADING=EAGER
for i in 1 2; do
mkdir -p /tmp/rep$i
( time MCRDL_MASTER_PORT=2966$i timeout 600 python tests/gpu_worker.py --threads 2 /tmp/rep$i golden,all_reduce,all_to_allv,all_to_all,gathers ) > gpurun_out/co5_$i.log 2>&1
python -c "
import json
for r in range(2):
    d=json.load(open('/tmp/rep$i/r%d.json'%r)); print(r, d['checked'], len(d['failures'])); [print('  ', f[:300]) for f in d['failures'][:3]]
" >> gpurun_out/co5_$i.log
grep -v "^   *[0-9]" gpurun_out/co5_$i.log | head -40
done
