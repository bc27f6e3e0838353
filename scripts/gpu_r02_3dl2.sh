#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/l2_3d.txt
: > $out
for v in "" "OOC_SWEEP_L2AHEAD=2" "OOC_SWEEP_L2AHEAD=4" "OOC_SWEEP_L2AHEAD=8" "OOC_SWEEP_L2AHEAD=4 OOC_SWEEP_P=2" "OOC_SWEEP_L2AHEAD=6 OOC_SWEEP_RB=14 OOC_SWEEP_P=1"; do
  env $v timeout 600 python scripts/sweep_time.py 600 3 miniflow3d >> $out 2>&1
  env $v timeout 600 python scripts/sweep_time.py 512 3 rk3chain3d >> $out 2>&1
done
OOC_SWEEP_L2AHEAD=4 timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q -m gpu -k "3d" > gpurun_out/l2_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/l2_pytest.log
