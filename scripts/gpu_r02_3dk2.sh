#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/k2_3d.txt
: > $out
for v in "" "OOC_SWEEP_K=2 OOC_SWEEP_P=1" "OOC_SWEEP_K=2 OOC_SWEEP_P=1 OOC_SWEEP_RB=12" "OOC_SWEEP_K=2 OOC_SWEEP_P=2"; do
  env $v timeout 600 python scripts/sweep_time.py 600 3 miniflow3d >> $out 2>&1
  env $v timeout 600 python scripts/sweep_time.py 512 3 rk3chain3d >> $out 2>&1
done
