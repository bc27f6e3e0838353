#!/bin/bash
# 3-D evidence at the final kernels: labelled launch lists (miniflow3d 600^3, rk3chain3d
# 512^3) and one full capture of the miniflow3d timestep sweep.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in "600 miniflow3d" "512 rk3chain3d"; do
  set -- $spec
  python scripts/ncu_driver.py $1 1 3 $2 > gpurun_out/ncu_driver_$2.log 2>&1 && cp gpurun_out/ncu_seq.json gpurun_out/ncu_seq_$2.json && cp gpurun_out/ncu_sweep_report.json gpurun_out/ncu_sweep_report_$2.json && \
  OOC_JIT_TUNE=gpurun_out/ncu_tune.txt timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02f_launches_$2.csv python scripts/ncu_driver.py $1 1 3 $2 > gpurun_out/ncu_launches_$2.log 2>&1
done
export OOC_SWEEP_P=3
python scripts/ncu_driver.py 600 1 2 miniflow3d > gpurun_out/ncu_driver_3dfull.log 2>&1 && \
OOC_JIT_TUNE=gpurun_out/ncu_tune.txt timeout 900 ncu --set full --clock-control none --import-source on -k regex:ooc_sweep_kernel --launch-skip 12 -c 1 -f -o gpurun_out/r02f_sweep3d_full python scripts/ncu_driver.py 600 1 2 miniflow3d > gpurun_out/ncu_full_3d.log 2>&1
echo done
