#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/kernel_sweep.py 7680 3 1x4,1x2,2x2,4x2,2x4,8x1 > gpurun_out/sweep_shapes.log 2>&1
python scripts/ncu_driver.py 7680 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ooc_jit -s 8 -c 6 -o gpurun_out/prof_fused python scripts/ncu_driver.py 7680 1 > gpurun_out/ncu_fused.log 2>&1
python scripts/ncu_driver.py 7680 0 > gpurun_out/plain0.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ooc_jit -s 28 -c 14 -o gpurun_out/prof_unfused python scripts/ncu_driver.py 7680 0 > gpurun_out/ncu_unfused.log 2>&1
echo done
