#!/bin/bash
# pytest -m gpu with the shipped exchange geometry, then chunk 128 vs 256 KiB at p = 2 and 4
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/xgeo_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/xgeo_pytest.log
for N in 2 4; do
  for C in 128 256; do
    MCRDL_X_CHUNK_KB=$C timeout 300 python -m torch.distributed.run --nnodes 1 \
      --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29581 -m paper_2303_08374_b200.tuner \
      --ops all_to_allv,all_gatherv --sizes 1M,4M,16M,64M,256M,1G --iters 20 --warmup 3 \
      2>/dev/null | grep "^all_" | sed "s/^/chunk=${C}K /"
  done
done > gpurun_out/xgeo_confirm.log 2>&1
