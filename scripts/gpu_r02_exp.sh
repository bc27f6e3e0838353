#!/bin/bash
# Sweep variants: 2 rows per step (2-D), ring lengths and tile rows (3-D).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "OOC_SWEEP_K=2 OOC_SWEEP_P=2" "OOC_SWEEP_K=2 OOC_SWEEP_P=1"; do
  tag=$(echo $v | tr ' =' '_-')
  env $v timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/r02x_bench_$tag.json 2> gpurun_out/r02x_bench_$tag.err
done
for v in "OOC_SWEEP_DEF=1" "OOC_SWEEP_RING=period" "OOC_SWEEP_RB=8"; do
tag=$(echo $v | tr ' =' '_-')
env $v python - > gpurun_out/r02x_3d_$tag.jsonl 2> gpurun_out/r02x_3d_$tag.err <<'PY'
import json, os, sys
sys.path.insert(0, os.getcwd())
import paper_1709_02125_b200 as B
def run(app, n, per, span):
    rt = B.Runtime("resident")
    rt.declare_app(app, n, n, n, span)
    rt.app_iterations(app, n, n, n, 0, per * 4, span)
    rt.sync()
    r0 = rt.report(); m0 = rt.mark()
    rt.app_iterations(app, n, n, n, per * 4, per * 7, span)
    m1 = rt.mark(); rt.sync()
    dt = rt.elapsed(m0, m1); r1 = rt.report()
    out = {"app": app, "n": n, "GBps": (r1["total_bytes"] - r0["total_bytes"]) / dt / 1e9,
           "sweeps": rt.device()["sweep_launches"], "tuning": B.sweep_report()}
    rt.close()
    return out
for app, n, per, span in (("miniflow3d", 600, 10, 0), ("rk3chain3d", 700, 3, 3)):
    print(json.dumps(run(app, n, per, span)), flush=True)
PY
done
echo done
