#!/bin/bash
# Row-sweep schedule sweep (profiles/r01_sweep_tuning.md): bench.py in-core value for each
# "K P SMEM RC" tuple given on the command line (P "auto" = autotuned), plus the sweep
# parity tests under the first tuple.
#   gpurun -- bash scripts/gpu_sweep_tuning.sh "1 auto 57344 256" "1 3 57344 256" "2 2 65536 128"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
first=1
for cfg in "$@"; do set -- $cfg
  env_p=""; [ "$2" != "auto" ] && env_p="OOC_SWEEP_P=$2"
  tag="k$1p$2s$3rc$4"
  if [ $first = 1 ]; then
    env OOC_SWEEP_K=$1 $env_p OOC_SWEEP_SMEM=$3 OOC_SWEEP_RC=$4 timeout 900 python -m pytest tests/test_gpu_sweep.py -q -x \
      > gpurun_out/pytest_sweep_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sweep_$tag.log
    first=0
  fi
  env OOC_SWEEP_K=$1 $env_p OOC_SWEEP_SMEM=$3 OOC_SWEEP_RC=$4 timeout 300 python bench.py --steps 3 --warmup 3 \
    --no-e2e --no-cpu > gpurun_out/bench_$tag.json 2>&1
done
echo done
