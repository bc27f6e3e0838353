#!/bin/bash
# 3-D plane-tile sweeps (tensor-copy producer): parity, then configs 4/5 in-core with and
# without them.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONFAULTHANDLER=1
timeout 1200 python -m pytest tests/test_gpu_sweep.py -x -q -k "3d or random" > gpurun_out/r02h_pytest_sweep3d.log 2>&1; echo "rc=$?" >> gpurun_out/r02h_pytest_sweep3d.log
python - > gpurun_out/r02h_3d.jsonl 2> gpurun_out/r02h_3d.err <<'PY'
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import paper_1709_02125_b200 as B
def run(app, n, per, span, sweep3d):
    B.set_sweep_3d(sweep3d)
    rt = B.Runtime("resident")
    rt.declare_app(app, n, n, n, span)
    rt.app_iterations(app, n, n, n, 0, per * 4, span)
    rt.sync()
    r0 = rt.report(); m0 = rt.mark()
    rt.app_iterations(app, n, n, n, per * 4, per * 7, span)
    m1 = rt.mark(); rt.sync()
    dt = rt.elapsed(m0, m1); r1 = rt.report()
    out = {"app": app, "n": n, "sweep3d": sweep3d, "GBps": (r1["total_bytes"] - r0["total_bytes"]) / dt / 1e9,
           "sweeps": rt.device()["sweep_launches"], "tuning": B.sweep_report()}
    rt.close()
    return out
for app, n, per, span in (("miniflow3d", 600, 10, 0), ("rk3chain3d", 700, 3, 3)):
    for s3 in (False, True):
        print(json.dumps(run(app, n, per, span, s3)), flush=True)
PY
echo done
