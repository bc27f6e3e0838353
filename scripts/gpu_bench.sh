#!/bin/bash
# Full-size bench + reference arm + ncu launch list of the same command + one
# `--set full` capture of the dominant fused kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launches.log 2>&1
python scripts/ncu_driver.py 15360 > gpurun_out/ncu_driver.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ooc_jit_kernel --launch-skip 31 -c 4 -f -o gpurun_out/top_full python scripts/ncu_driver.py 15360 > gpurun_out/ncu_full.log 2>&1
echo done
