"""Experiment: in-core miniflow2d effective GB/s per kernel variant / fusion setting.
Usage: python scripts/kernel_sweep.py N STEPS  (each config in a fresh process)."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 7680
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
CHILD = r'''
import sys, json, os
sys.path.insert(0, %r)
import paper_1709_02125_b200 as B
n, steps, fuse = %d, %d, %d
rt = B.Runtime("resident", fuse=bool(fuse), profile=True)
rt.declare_app("miniflow2d", n, n)
rt.app_iterations("miniflow2d", n, n, 0, 0, 20)
rt.sync(); r0 = rt.report(); lm0 = {m[0] for m in rt.loop_metrics()}
m0 = rt.mark(); rt.app_iterations("miniflow2d", n, n, 0, 20, 20 + 10 * steps); m1 = rt.mark()
dt = rt.elapsed(m0, m1); r1 = rt.report()
lm = [m for m in rt.loop_metrics() if m[0] not in lm0]
first = min(m[0] for m in lm)
kinds = {}
for m in lm:
    p = (m[0] - first) %% 141
    k = "fieldsum" if p == 140 else "L%%d" %% (p %% 14 + 1)
    a = kinds.setdefault(k, [0, 0.0]); a[0] += m[2]; a[1] += m[3]
d = rt.device()
print(json.dumps({"n": n, "fuse": fuse, "jit": os.environ.get("OOC_JIT", ""), "shape": os.environ.get("OOC_JIT_SHAPE", ""), "jit_launches": d["jit_launches"], "jit_compile_ms": d["jit_compile_ms"],
                  "GBps": (r1["total_bytes"] - r0["total_bytes"]) / dt / 1e9,
                  "ms_per_step": 1e3 * dt / steps, "dev": rt.device()["kernel_launches"],
                  "per_loop_GBps": {k: round(v[0] / v[1] / 1e9) for k, v in sorted(kinds.items()) if v[1] > 0}}))
'''
shapes = sys.argv[3].split(",") if len(sys.argv) > 3 else [""]
for shape in shapes:
    for fuse in (1, 0):
        jit = "1"
        env = dict(os.environ, OOC_JIT=jit, OOC_JIT_SHAPE=shape)
        r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, n, steps, fuse)], env=env,
                           capture_output=True, text=True, timeout=600)
        print(r.stdout.strip() or r.stderr[-2000:], flush=True)
