#!/bin/bash
# Edge-first CTA order: CTA schedule trace, sweep parity tests, bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
OOC_GRAPHS=0 OOC_SWEEP_TRACE=gpurun_out/sweep_trace.txt timeout 600 python scripts/sweep_trace.py 15360 > gpurun_out/sweep_trace_summary.txt 2>&1
echo "rc=$?" >> gpurun_out/sweep_trace_summary.txt
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_parity_large.py -x -q -m gpu > gpurun_out/edge_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/edge_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-parity > gpurun_out/edge_bench.json 2> gpurun_out/edge_bench.err
echo "rc=$?" >> gpurun_out/edge_bench.err
OOC_SWEEP_MASKED=0 timeout 900 python bench.py --steps 5 --warmup 3 --no-parity > gpurun_out/edge0_bench.json 2> gpurun_out/edge0_bench.err
