#!/bin/bash
# Sweep-kernel variants (rows per step, ring width) + a source-level ncu capture of the TMA kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "OOC_SWEEP_K=2" "OOC_SWEEP_RC=128" "OOC_SWEEP_K=2 OOC_SWEEP_UNROLL=0" "OOC_SWEEP_TMA=1"; do
  tag=$(echo $v | tr ' =' '_-')
  env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r02b_bench_$tag.json 2> gpurun_out/r02b_bench_$tag.err
done
export OOC_SWEEP_P=3
python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_driver.log 2>&1 && \
OOC_JIT_TUNE=gpurun_out/ncu_tune.txt timeout 900 ncu --set full --clock-control none --import-source on -k regex:ooc_sweep_kernel --launch-skip 20 -c 1 -f -o gpurun_out/r02_sweep_tma python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_full.log 2>&1
echo done
