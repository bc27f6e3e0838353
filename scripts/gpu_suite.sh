#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 2400 python scripts/suite.py > gpurun_out/suite.jsonl 2> gpurun_out/suite.err; echo "suite rc=$?" >> gpurun_out/suite.err
