#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/fuzz.txt
: > $out
timeout 1500 python scripts/fuzz_sweeps.py 5000 60 >> $out 2>&1; echo "rc=$?" >> $out
OOC_SWEEP_RC=64 OOC_SWEEP_SMEM=60000 timeout 1500 python scripts/fuzz_sweeps.py 6000 60 >> $out 2>&1; echo "rc=$?" >> $out
OOC_SWEEP_RC=128 OOC_SWEEP_K=2 timeout 1500 python scripts/fuzz_sweeps.py 7000 40 >> $out 2>&1; echo "rc=$?" >> $out
