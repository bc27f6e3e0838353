#!/bin/bash
# Evidence C (after the sweep scheduling changes): whole GPU suite, smoke, bench, reference arm,
# labelled 2-D ncu launch list (generator-hash stamped) + one full capture of the sweep.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r02c_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02_smoke.log
timeout 1200 python bench.py > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; echo "bench rc=$?" >> gpurun_out/r02_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02c_bench_ref.json 2> gpurun_out/r02c_bench_ref.err
export OOC_SWEEP_P=4
python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_driver.log 2>&1 && \
OOC_JIT_TUNE=gpurun_out/ncu_tune.txt timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none --csv --log-file gpurun_out/r02c_launches.csv python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_launches.log 2>&1 && \
cp gpurun_out/ncu_sweep_report.json gpurun_out/ncu_sweep_report_2d.json && cp gpurun_out/ncu_seq.json gpurun_out/ncu_seq_2d.json && \
OOC_JIT_TUNE=gpurun_out/ncu_tune.txt timeout 900 ncu --set full --clock-control none --import-source on -k regex:ooc_sweep_kernel --launch-skip 20 -c 1 -f -o gpurun_out/r02c_sweep_full python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_full.log 2>&1
echo done
