#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 900 python -m pytest tests/test_gpu_sweep.py "tests/test_gpu_parity.py::test_slab_runtime_with_nccl_single_rank" "tests/test_gpu_parity.py::test_graph_replay_parity" -q -x > gpurun_out/pytest_sweep.log 2>&1; echo "sweep rc=$?" >> gpurun_out/pytest_sweep.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
echo done
