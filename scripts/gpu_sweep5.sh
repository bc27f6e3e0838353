#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
OOC_SWEEP_K=1 OOC_SWEEP_P=1 OOC_SWEEP_SMEM=40000 timeout 900 python -m pytest tests/test_gpu_sweep.py -q -x > gpurun_out/pytest_sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/pytest_sweep.log
for k in "1 1 34000" "1 1 56000" "1 1 74000" "2 1 40000" "2 1 56000" "1 2 40000" "2 2 56000" "4 1 80000"; do set -- $k
OOC_SWEEP_K=$1 OOC_SWEEP_P=$2 OOC_SWEEP_SMEM=$3 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_k$1p$2s$3.json 2>&1
done
echo done
