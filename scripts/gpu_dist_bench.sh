#!/bin/bash
# The bench's slab (multi-GPU) path on one GPU: torchrun, one rank, NCCL communicator,
# ghost exchange + all-reduce per chain (OOC_BENCH_FORCE_DIST=1); plus the reference arm
# launched the way the driver's scaling run launches it.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533"
OOC_BENCH_FORCE_DIST=1 timeout 900 $TR bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/dist_bench.json 2> gpurun_out/dist_bench.err; echo "rc=$?" >> gpurun_out/dist_bench.err
timeout 600 $TR bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/dist_ref.json 2> gpurun_out/dist_ref.err; echo "rc=$?" >> gpurun_out/dist_ref.err
echo done
