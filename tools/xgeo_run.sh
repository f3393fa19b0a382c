#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/xgeo_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/xgeo_pytest.log
bash tools/xgeo_ab.sh 4 > gpurun_out/xgeo_ab_p4.log 2>&1
