#!/bin/bash
# L2-prefetch variants of the sweep, BASELINE configs 2-5 + high-reuse span-10 chains, and
# labelled ncu launch lists of the 3-D apps.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
for v in "OOC_SWEEP_L2AHEAD=4" "OOC_SWEEP_L2AHEAD=12"; do
  tag=$(echo $v | tr ' =' '_-')
  env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r02f_bench_$tag.json 2> gpurun_out/r02f_bench_$tag.err
done
timeout 3600 python scripts/suite.py 2 3 4 5 5s10 2s10 > gpurun_out/r02_suite.jsonl 2> gpurun_out/r02_suite.err; echo "suite rc=$?" >> gpurun_out/r02_suite.err
for spec in "600 miniflow3d" "512 rk3chain3d"; do
  set -- $spec
  python scripts/ncu_driver.py $1 1 3 $2 > gpurun_out/ncu_driver_$2.log 2>&1 && cp gpurun_out/ncu_seq.json gpurun_out/ncu_seq_$2.json && \
  OOC_JIT_TUNE=gpurun_out/ncu_tune.txt timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_$2.csv python scripts/ncu_driver.py $1 1 3 $2 > gpurun_out/ncu_launches_$2.log 2>&1
done
echo done
