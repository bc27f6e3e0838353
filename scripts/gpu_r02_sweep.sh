#!/bin/bash
# Round-2 sweep kernel check: parity tests of the row sweeps, then in-core bench variants.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q > gpurun_out/r02_pytest_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/r02_pytest_sweep.log
for v in "OOC_SWEEP_TMA=1" "OOC_SWEEP_TMA=0" "OOC_SWEEP_UNROLL=0" "OOC_SWEEP_TMA=0 OOC_SWEEP_UNROLL=0"; do
  env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02_bench_$(echo $v | tr ' =' '_-').json 2> gpurun_out/r02_bench_$(echo $v | tr ' =' '_-').err
done
echo done
