#!/bin/bash
# Final check at HEAD: whole GPU suite + smoke (2-D kernels unchanged since r02_final_*).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r02d_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02d_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02d_smoke.log
timeout 1200 python bench.py > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo "rc=$?" >> gpurun_out/r02d_bench.err
