#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OOC_GRAPHS=0 OOC_SWEEP_TRACE=gpurun_out/t3d_off.txt timeout 600 python scripts/sweep_trace.py 600 miniflow3d > /dev/null 2>&1
OOC_SWEEP_MASKED3=1 OOC_GRAPHS=0 OOC_SWEEP_TRACE=gpurun_out/t3d_on.txt timeout 600 python scripts/sweep_trace.py 600 miniflow3d > /dev/null 2>&1
echo done
