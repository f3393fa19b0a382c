#!/bin/bash
# usage: tools/sweep.sh NGPU TAG [tuner args...]  (run on the GPU box)
N=$1; TAG=$2; shift 2
python -m torch.distributed.run --nnodes 1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  -m paper_2303_08374_b200.tuner --csv gpurun_out/sweep_${TAG}.csv "$@" > gpurun_out/sweep_${TAG}.log 2>&1
echo "sweep rc=$?"
