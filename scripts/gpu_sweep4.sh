#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for k in "2 1 56000" "2 1 74000" "2 1 110000" "4 1 56000" "4 1 74000" "4 1 110000" "1 1 40000" "1 1 56000" "2 2 74000"; do set -- $k
OOC_SWEEP_K=$1 OOC_SWEEP_P=$2 OOC_SWEEP_SMEM=$3 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_k$1p$2s$3.json 2>&1
done
echo done
