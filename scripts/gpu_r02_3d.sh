#!/bin/bash
# 3-D plane-tile sweeps: parity (2-D regression + 3-D), in-core 2-D bench, configs 4/5.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests/test_gpu_sweep.py -x -q > gpurun_out/r02g_pytest_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r02g_pytest_sweep.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
timeout 2400 python scripts/suite.py 4 5 > gpurun_out/r02g_suite45.jsonl 2> gpurun_out/r02g_suite45.err; echo "rc=$?" >> gpurun_out/r02g_suite45.err
echo done
