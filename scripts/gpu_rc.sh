#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for rc in 256 64; do
OOC_SWEEP_RC=$rc timeout 900 python -m pytest tests/test_gpu_sweep.py -q -x -k "apps or random" > gpurun_out/pytest_rc$rc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rc$rc.log
OOC_SWEEP_RC=$rc timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_rc$rc.json 2>&1
done
OOC_SWEEP_RC=256 OOC_SWEEP_P=2 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_rc256p2.json 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_rc128.json 2>&1
echo done
