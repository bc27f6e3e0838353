"""Small, deterministic driver for ncu captures: miniflow2d resident, `chains`
10-iteration chains (the first ones compile + tune every fused kernel). Writes the
launch sequence of the last chain — (first loop position, loops) per launch — to
gpurun_out/ncu_seq.json so scripts/ncu_summarize.py can label ncu's launch list.

    python scripts/ncu_driver.py [n] [fuse] [chains] [app]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1709_02125_b200 as B  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 15360
fuse = int(sys.argv[2]) if len(sys.argv) > 2 else 1
chains = int(sys.argv[3]) if len(sys.argv) > 3 else 3
app = sys.argv[4] if len(sys.argv) > 4 else "miniflow2d"
nz = n if app.endswith("3d") else 0
rt = B.Runtime("resident", fuse=bool(fuse), profile=True)
rt.declare_app(app, n, n, nz)
for c in range(chains):
    first_id = max((m[0] for m in rt.loop_metrics()), default=-1) + 1
    rt.app_iterations(app, n, n, nz, 10 * c, 10 * (c + 1))
    rt.sync()
    log = rt.launch_log()
seq = [[first - first_id, nl, nbytes] for first, nl, nbytes, _ in log]
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
seq_name = "ncu_seq.json" if not os.environ.get("OOC_JIT_TUNE") else "ncu_seq_replay.json"
with open(os.path.join(ROOT, "gpurun_out", seq_name), "w") as f:
    json.dump({"app": app, "n": n, "fuse": fuse, "chains": chains, "last_chain": seq}, f)
with open(os.path.join(ROOT, "gpurun_out", "ncu_sweep_report.json"), "w") as f:
    json.dump(B.sweep_report(), f)  # generator hashes of the sweep kernels this run built
with open(os.path.join(ROOT, "gpurun_out", "ncu_tune.txt"), "w") as f:
    for k in B.jit_report():  # replay these shapes under ncu: OOC_JIT_TUNE=gpurun_out/ncu_tune.txt
        if k["shape"]:
            f.write(f"{k['key']} {k['shape']}\n")
print(rt.device())
