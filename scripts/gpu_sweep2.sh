#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_sweep.py -q -x > gpurun_out/pytest_sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/pytest_sweep.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
for k in "2 2" "4 1" "4 2" "1 2" "8 1"; do set -- $k
OOC_SWEEP_K=$1 OOC_SWEEP_P=$2 OOC_SWEEP_SMEM=200000 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_k$1p$2_big.json 2>&1
OOC_SWEEP_K=$1 OOC_SWEEP_P=$2 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_k$1p$2.json 2>&1
done
echo done
