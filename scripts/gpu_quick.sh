#!/bin/bash
# pytest -m gpu + bench (no reference arm) + labelled ncu launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_driver.log 2>&1 && \
OOC_JIT_TUNE=gpurun_out/ncu_tune.txt timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_launches.log 2>&1
echo done
