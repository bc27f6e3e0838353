#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python scripts/e2e_sweep.py > gpurun_out/e2e_sweep.log 2>&1; echo "e2e rc=$?" >> gpurun_out/e2e_sweep.log
timeout 1800 python scripts/suite.py 2 4 5 > gpurun_out/suite2.jsonl 2> gpurun_out/suite2.err; echo "suite rc=$?" >> gpurun_out/suite2.err
echo done
