#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/mask2.txt
: > $out
for m in 1 2; do
  OOC_SWEEP_MASKED=$m OOC_GRAPHS=0 OOC_SWEEP_TRACE=gpurun_out/t2d_m$m.txt timeout 600 python scripts/sweep_trace.py 15360 > gpurun_out/t2d_m${m}_summary.txt 2>&1
  OOC_SWEEP_MASKED=$m timeout 900 python bench.py --steps 5 --warmup 3 --no-parity --no-cpu > gpurun_out/mask2_bench_$m.json 2>/dev/null
done
OOC_SWEEP_MASKED=2 timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q -m gpu > gpurun_out/mask2_pytest.log 2>&1; echo rc=$? >> gpurun_out/mask2_pytest.log
