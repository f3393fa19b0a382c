set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1z_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1z_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1z_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r1z_bench_n1.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/r1z_ref_n1.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r1z_bench_n4.log 2>&1
tail -n 3 gpurun_out/r1z_*.log
