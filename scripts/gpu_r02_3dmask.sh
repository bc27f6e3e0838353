#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/mask_3d.txt
: > $out
for v in "" "OOC_SWEEP_MASKED=0"; do
  env $v timeout 600 python scripts/sweep_time.py 600 3 miniflow3d >> $out 2>&1
  env $v timeout 600 python scripts/sweep_time.py 512 3 rk3chain3d >> $out 2>&1
done
timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q -m gpu -k "3d" > gpurun_out/mask_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/mask_pytest.log
