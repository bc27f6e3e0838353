#!/bin/bash
# Round-2 evidence: bench (parity leg, CPU baselines), reference arm, labelled ncu launch
# list with DRAM bytes (generator-hash stamped), one --set full capture of the sweep kernel,
# large-size parity tests and the two-ranks-on-one-GPU bench test.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
{ nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/r02_clocks.csv & } ; CLK=$!
timeout 1200 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?" >> gpurun_out/r02_bench.err
kill $CLK
timeout 600 python bench.py --impl reference > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err
timeout 1200 python -m pytest tests/test_gpu_parity_large.py "tests/test_bench_contract.py::test_bench_two_ranks_on_one_gpu_decompose_one_mesh" -q -x > gpurun_out/r02_pytest_large.log 2>&1; echo "rc=$?" >> gpurun_out/r02_pytest_large.log
export OOC_SWEEP_P=4
python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_driver.log 2>&1 && \
OOC_JIT_TUNE=gpurun_out/ncu_tune.txt timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_launches.log 2>&1 && \
OOC_JIT_TUNE=gpurun_out/ncu_tune.txt timeout 900 ncu --set full --clock-control none --import-source on -k regex:ooc_sweep_kernel --launch-skip 20 -c 1 -f -o gpurun_out/r02_sweep_full python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_full.log 2>&1
echo done
