#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q > gpurun_out/r02c_pytest_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r02c_pytest_sweep.log
for v in "OOC_SWEEP_SKEW=1" "OOC_SWEEP_SKEW=0"; do
  tag=$(echo $v | tr ' =' '_-')
  env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r02c_bench_$tag.json 2> gpurun_out/r02c_bench_$tag.err
done
echo done
