#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
OOC_ROW_RECOMPUTE=1 OOC_JIT_SHAPE=t8x128w512 timeout 300 python tests/shape_parity_child.py > gpurun_out/child_rc.log 2>&1; echo "child rc=$?" >> gpurun_out/child_rc.log
OOC_ROW_RECOMPUTE=1 timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_rc.json 2> gpurun_out/bench_rc.err; echo "rc=$?" >> gpurun_out/bench_rc.err
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
echo done
