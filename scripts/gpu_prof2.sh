#!/bin/bash
# K/P variants with forwarding + the ncu evidence of the default configuration.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "2 1 48000 0" "2 1 64000 0" "4 1 64000 0" "4 1 96000 0" "2 2 64000 0" "1 2 48000 0"; do set -- $cfg
OOC_SWEEP_K=$1 OOC_SWEEP_P=$2 OOC_SWEEP_SMEM=$3 OOC_SWEEP_MINB=$4 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_k$1p$2s$3m$4.json 2>&1
done
python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_driver.log 2>&1 && \
OOC_JIT_TUNE=gpurun_out/ncu_tune.txt timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_launches.log 2>&1
OOC_JIT_TUNE=gpurun_out/ncu_tune.txt timeout 900 ncu --set full --clock-control none --import-source on -k regex:ooc_sweep_kernel --launch-skip 20 -c 1 -f -o gpurun_out/sweep_full python scripts/ncu_driver.py 15360 1 3 > gpurun_out/ncu_full.log 2>&1
echo done
