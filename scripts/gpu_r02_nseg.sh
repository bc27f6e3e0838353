#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/nseg.txt
: > $out
for ns in 0 29 40 48 60 75 90 120; do
  OOC_SWEEP_NSEG=$ns timeout 300 python scripts/sweep_time.py 15360 4 >> $out 2>&1
done
