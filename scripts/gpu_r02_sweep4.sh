#!/bin/bash
# Period rings (non-power-of-two lengths) + L2 prefetch: parity, then in-core variants.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q > gpurun_out/r02d_pytest_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r02d_pytest_sweep.log
for v in "OOC_SWEEP_DEF=1" "OOC_SWEEP_P=1" "OOC_SWEEP_P=2" "OOC_SWEEP_L2AHEAD=0" "OOC_SWEEP_RING=pow2" "OOC_SWEEP_L2AHEAD=8"; do
  tag=$(echo $v | tr ' =' '_-')
  env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r02d_bench_$tag.json 2> gpurun_out/r02d_bench_$tag.err
done
echo done
