#!/bin/bash
# New round-2 GPU tests first (IPC slabs on one GPU, reference apps.cpp on this runtime,
# executor seam), then the whole GPU suite, then smoke.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests/test_gpu_dist_ipc.py tests/test_gpu_native_api.py -x -q -m gpu > gpurun_out/r02_pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/r02_pytest_new.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r02_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02_smoke.log
echo done
