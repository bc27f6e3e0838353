#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reports.py tests/test_gpu_native_api.py -q -x > gpurun_out/pytest_ooc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ooc.log
timeout 900 python scripts/suite.py 3 4 5 > gpurun_out/suite_ooc.jsonl 2> gpurun_out/suite_ooc.err
timeout 400 python scripts/timeline_dump.py miniflow3d 600 600 600 50 3 > gpurun_out/timeline3d.log 2>&1
echo done
