#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/ab_3d.txt
: > $out
for v in "" "OOC_SWEEP_EDGEFIRST=0" "OOC_SWEEP_MASKED=0" "OOC_SWEEP_NSEG_OLD=1" "OOC_SWEEP_EDGEFIRST=0 OOC_SWEEP_MASKED=0 OOC_SWEEP_NSEG_OLD=1"; do
  env $v OOC_SWEEP_DEBUG=1 timeout 600 python scripts/sweep_time.py 600 3 miniflow3d >> $out 2>gpurun_out/ab_3d_dbg.txt
  tail -2 gpurun_out/ab_3d_dbg.txt >> $out
done
OOC_GRAPHS=0 OOC_SWEEP_TRACE=gpurun_out/sweep_trace3d.txt timeout 600 python scripts/sweep_trace.py 600 miniflow3d > gpurun_out/sweep_trace3d_summary.txt 2>&1
