#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/knobs_3d.txt
: > $out
for v in "" "OOC_SWEEP_K=2" "OOC_SWEEP_RB=8" "OOC_SWEEP_RB=24" "OOC_SWEEP_RC3=64 OOC_SWEEP_RB=8" "OOC_SWEEP_RING=period" "OOC_SWEEP_P=2" "OOC_SWEEP_P=4" "OOC_SWEEP_UNROLL=0"; do
  env $v timeout 600 python scripts/sweep_time.py 600 3 miniflow3d >> $out 2>&1
done
