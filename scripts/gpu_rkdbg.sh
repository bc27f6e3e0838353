#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for sm in 48000 30000; do
OOC_SWEEP_SMEM=$sm timeout 120 python scripts/sweep_rk_child.py rk3chain 200 256 6 3 >> gpurun_out/rkdbg.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_sweep.py -q -x > gpurun_out/pytest_sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/pytest_sweep.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_default.json 2>&1
OOC_SWEEP_MINB=6 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_minb6.json 2>&1
echo done
