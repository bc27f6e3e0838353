#!/bin/bash
# Round-end evidence run: GPU tests, smoke, bench (+ reference arm), BASELINE configs
# 2-5, measured OOC timeline, labelled ncu launch list (tuning replayed), and one
# `--set full` capture of the dominant kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 1500 python scripts/suite.py > gpurun_out/suite.jsonl 2> gpurun_out/suite.err
timeout 400 python scripts/timeline_dump.py miniflow2d 15360 15360 0 50 3 > gpurun_out/timeline2d.log 2>&1
timeout 400 python scripts/timeline_dump.py miniflow3d 600 600 600 50 3 > gpurun_out/timeline3d.log 2>&1
python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_driver.log 2>&1 && \
OOC_JIT_TUNE=gpurun_out/ncu_tune.txt timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_launches.log 2>&1 && \
OOC_JIT_TUNE=gpurun_out/ncu_tune.txt timeout 900 ncu --set full --clock-control none --import-source on -k regex:ooc_sweep_kernel --launch-skip 20 -c 1 -f -o gpurun_out/top_full python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_full.log 2>&1
echo done
