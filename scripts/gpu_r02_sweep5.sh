#!/bin/bash
# Lane-parallel producer: parity, then budget / prefetch variants.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q > gpurun_out/r02e_pytest_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r02e_pytest_sweep.log
for v in "OOC_SWEEP_DEF=1" "OOC_SWEEP_SMEM=80000" "OOC_SWEEP_SMEM=80000 OOC_SWEEP_L2AHEAD=0" "OOC_SWEEP_SMEM=100000" "OOC_SWEEP_RING=pow2 OOC_SWEEP_L2AHEAD=0"; do
  tag=$(echo $v | tr ' =' '_-')
  env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r02e_bench_$tag.json 2> gpurun_out/r02e_bench_$tag.err
done
echo done
