cd $GRAFT_REPO_ROOT
timeout 400 python tests/gpu_launch.py 4 baseline,pool > gpurun_out/t3_p4.log 2>&1; echo p4 rc=$?; head -5 gpurun_out/t3_p4.log
MCRDL_LAUNCH_TIMEOUT=350 timeout 400 python tests/gpu_launch.py 2 baseline --colocated > gpurun_out/t3_co2.log 2>&1; echo co2 rc=$?; head -3 gpurun_out/t3_co2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29504 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/t3_bench_n4.log 2>&1; echo "bench n4 rc=$?"
python -c "
import json
l=[x for x in open('gpurun_out/t3_bench_n4.log') if x.startswith('{')][-1]; d=json.loads(l)
print(d['value'], d['mixed_step_cfg5'], d.get('all_reduce_symmetric'))
"
