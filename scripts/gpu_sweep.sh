#!/bin/bash
# Row-sweep kernels: parity first, then the full GPU suite and the bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_sweep.py -q -x > gpurun_out/pytest_sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/pytest_sweep.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done
