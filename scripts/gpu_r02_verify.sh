#!/bin/bash
# Round-2 final verification at HEAD: whole GPU suite, smoke, default bench, reference arm.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r02v_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02v_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02v_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02v_smoke.log
timeout 1200 python bench.py > gpurun_out/r02v_bench.json 2> gpurun_out/r02v_bench.err; echo "bench rc=$?" >> gpurun_out/r02v_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02v_bench_ref.json 2> gpurun_out/r02v_bench_ref.err
echo done
