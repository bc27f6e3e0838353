#!/bin/bash
# Sweep changes: parity (sweep + large), 3-D timings with/without the new scheduling, bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/check_3d.txt
: > $out
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_parity_large.py -x -q -m gpu > gpurun_out/check_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/check_pytest.log
for app in miniflow3d rk3chain3d; do
  n=600; [ $app = rk3chain3d ] && n=512
  timeout 600 python scripts/sweep_time.py $n 3 $app >> $out 2>&1
  OOC_SWEEP_EDGEFIRST=0 OOC_SWEEP_MASKED=0 OOC_SWEEP_NSEG_OLD=1 timeout 600 python scripts/sweep_time.py $n 3 $app >> $out 2>&1
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-parity > gpurun_out/check_bench.json 2> gpurun_out/check_bench.err
echo "rc=$?" >> gpurun_out/check_bench.err
