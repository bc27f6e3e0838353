#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export OOC_SWEEP_P=3 OOC_SWEEP_3D=1
python scripts/ncu_driver.py 400 1 2 miniflow3d > gpurun_out/ncu_driver_3d.log 2>&1 && \
OOC_JIT_TUNE=gpurun_out/ncu_tune.txt timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_mf3d_sweep.csv python scripts/ncu_driver.py 400 1 2 miniflow3d > gpurun_out/ncu_launches_3d.log 2>&1 && \
OOC_JIT_TUNE=gpurun_out/ncu_tune.txt timeout 900 ncu --set full --clock-control none --import-source on -k regex:ooc_sweep_kernel --launch-skip 12 -c 1 -f -o gpurun_out/r02_sweep3d_full python scripts/ncu_driver.py 400 1 2 miniflow3d > gpurun_out/ncu_full_3d.log 2>&1
echo done
