#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_sweep.py -q -x -k "apps or random or graph" > gpurun_out/pytest_sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/pytest_sweep.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_restrict.json 2>&1
OOC_SWEEP_RESTRICT=0 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_norestrict.json 2>&1
echo done
