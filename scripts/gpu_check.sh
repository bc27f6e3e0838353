#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python scripts/kernel_sweep.py 7680 3 > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/sweep.log
timeout 600 python scripts/kernel_sweep.py 15360 3 > gpurun_out/sweep15k.log 2>&1; echo "sweep rc=$?" >> gpurun_out/sweep15k.log
timeout 300 python bench.py --n 3840 --steps 2 --warmup 1 --no-e2e > gpurun_out/bench_cpu.log 2> gpurun_out/bench_cpu.err; echo "bench-cpu rc=$?" >> gpurun_out/bench_cpu.log
