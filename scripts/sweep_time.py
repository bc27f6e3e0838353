"""Median device time of the miniflow2d timestep sweep launches (14 loops), resident,
profiled launches (CUDA events around each launch). Prints one line per run.

    python scripts/sweep_time.py [n] [chains] [app]
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1709_02125_b200 as B  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 15360
chains = int(sys.argv[2]) if len(sys.argv) > 2 else 4
app = sys.argv[3] if len(sys.argv) > 3 else "miniflow2d"
nz = n if app.endswith("3d") else 0
rt = B.Runtime("resident", profile=True)
rt.declare_app(app, n, n, nz)
for c in range(chains):
    rt.app_iterations(app, n, n, nz, 10 * c, 10 * (c + 1))
    rt.sync()
    log = rt.launch_log()
by = {}
for first, nl, nbytes, sec in log:
    by.setdefault(nl, []).append(sec)
env = {k: v for k, v in os.environ.items() if k.startswith("OOC_")}
print(env, {nl: (len(v), round(statistics.median(v) * 1e3, 4)) for nl, v in sorted(by.items())}, flush=True)
