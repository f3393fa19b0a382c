#!/bin/bash
# parity with the shipped exchange geometry
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/xgeo_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/xgeo_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/xgeo_pytest.log 2>&1
