#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_parity.py -x -q -m gpu -k "3d or medium or golden" > gpurun_out/smem3_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/smem3_pytest.log
out=gpurun_out/smem3_time.txt
: > $out
timeout 600 python scripts/sweep_time.py 512 3 rk3chain3d >> $out 2>&1
timeout 600 python scripts/sweep_time.py 700 2 rk3chain3d >> $out 2>&1
OOC_SWEEP_SMEM3=204800 timeout 600 python scripts/sweep_time.py 700 2 rk3chain3d >> $out 2>&1
timeout 600 python scripts/sweep_time.py 600 3 miniflow3d >> $out 2>&1
