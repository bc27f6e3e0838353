#!/bin/bash
# Round-2 baseline: host facts + a source-level ncu capture of the current row-sweep kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ free -g; nproc; lscpu | grep -iE 'numa|model name|socket'; nvidia-smi topo -m; cat /sys/class/drm/*/device/numa_node 2>/dev/null | head -3; } > gpurun_out/host.txt 2>&1
export OOC_SWEEP_P=3
python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_driver.log 2>&1 && \
OOC_JIT_TUNE=gpurun_out/ncu_tune.txt timeout 900 ncu --set full --clock-control none --import-source on -k regex:ooc_sweep_kernel --launch-skip 20 -c 1 -f -o gpurun_out/r02_sweep_base python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_full.log 2>&1
echo done
