#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_sweep.py -q -x > gpurun_out/pytest_sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/pytest_sweep.log
for k in "2 2 110000" "4 2 110000" "4 1 110000" "2 1 110000" "2 2 200000" "4 2 200000" "8 1 200000" "1 2 110000"; do set -- $k
OOC_SWEEP_K=$1 OOC_SWEEP_P=$2 OOC_SWEEP_SMEM=$3 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_k$1p$2s$3.json 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ooc_sweep_kernel --launch-skip 8 -c 1 -f -o gpurun_out/sweep_full python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_sweep.log 2>&1
echo done
