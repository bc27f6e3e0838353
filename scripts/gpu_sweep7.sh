#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_sweep.py -q -x > gpurun_out/pytest_sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/pytest_sweep.log
for cfg in "1 1 48000 0" "1 1 48000 5" "1 1 48000 6" "2 1 48000 0" "2 1 60000 0" "1 1 74000 0" "2 1 74000 4"; do set -- $cfg
OOC_SWEEP_K=$1 OOC_SWEEP_P=$2 OOC_SWEEP_SMEM=$3 OOC_SWEEP_MINB=$4 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_k$1p$2s$3m$4.json 2>&1
done
echo done
