#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./scripts/probes/copy_probe > gpurun_out/copy_probe.txt 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_default.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ooc_sweep_kernel --launch-skip 20 -c 1 -f -o gpurun_out/sweep_full python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_sweep.log 2>&1
echo done
