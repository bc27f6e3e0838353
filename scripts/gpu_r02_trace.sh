#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OOC_GRAPHS=0 OOC_SWEEP_TRACE=gpurun_out/sweep_trace.txt timeout 600 python scripts/sweep_trace.py 15360 > gpurun_out/sweep_trace_summary.txt 2>&1
echo "rc=$?" >> gpurun_out/sweep_trace_summary.txt
