#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python scripts/kernel_sweep.py 7680 3 1x4,2x4,1x8,4x2,2x2,1x2 > gpurun_out/sweep_shapes.log 2>&1
echo done
