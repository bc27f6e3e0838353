#!/bin/bash
# TMA template bring-up: forced-shape parity, then a bench and a labelled launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for sh in t16x64 t8x128; do
  OOC_JIT_SHAPE=$sh timeout 300 python tests/shape_parity_child.py > gpurun_out/tma_$sh.log 2>&1; echo "rc=$?" >> gpurun_out/tma_$sh.log
done
OOC_JIT_SHAPE=t16x64 OOC_ROW_RECOMPUTE=1 timeout 300 python tests/shape_parity_child.py > gpurun_out/tma_rc.log 2>&1; echo "rc=$?" >> gpurun_out/tma_rc.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
OOC_ROW_RECOMPUTE=1 timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench_rc.json 2> gpurun_out/bench_rc.err
echo done
