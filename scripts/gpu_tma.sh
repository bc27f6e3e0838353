#!/bin/bash
# TMA template: bench (autotuned among register + TMA shapes), row recompute variant,
# labelled launch lists.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
OOC_ROW_RECOMPUTE=1 timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_rc.json 2> gpurun_out/bench_rc.err; echo "rc=$?" >> gpurun_out/bench_rc.err
OOC_JIT_SHAPE=t16x64 timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_t16.json 2> gpurun_out/bench_t16.err
OOC_ROW_RECOMPUTE=1 OOC_JIT_SHAPE=t16x64 timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_rc_t16.json 2> gpurun_out/bench_rc_t16.err
echo done
