"""One rank of a slab-decomposed run over the CUDA-IPC transport (tests/test_gpu_dist_ipc.py).

    python tests/dist_ipc_child.py <rank> <world> <name> <executor> <app> <nx> <ny> <nz> <iters> <span> <out.npz>

Runs the app on this rank's dim-0 slab with the product's kernels and exchanges, then
saves its owned rows (plus the global edge rows at the first/last rank) of every
dataset, their stale flags and the reductions.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1709_02125_b200 as B  # noqa: E402
from paper_1709_02125_b200 import dist as D  # noqa: E402

rank, world, name, executor, app = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], sys.argv[5]
nx, ny, nz, iters, span = (int(x) for x in sys.argv[6:11])
out = sys.argv[11]
cyclic = os.environ.get("OOC_TEST_CYCLIC") == "1"
B.set_jit(2, 0)  # specialised kernels (row sweeps for resident 2-D chains) at test sizes
nd = 3 if nz else 2
ghost = D.chain_depth(app, iters, span, nd)
pad = 3 * (span or 1) - 1 if app.startswith("rk3") else 0
own = D.slab(rank, world, nx + 2 * pad, -pad)
kw = dict(dist=(rank, world), own=own, ghost=ghost, gpu=0)
if executor == "explicit":
    # each rank streams its own slab through 3 HBM slots in 3 skewed tiles
    rt = B.Runtime("explicit", tiles=3, prefetch=True, **kw)
else:
    rt = B.Runtime("resident", **kw)
rt.comm_init_ipc(name)
rt.run_app(app, nx, ny, nz, iters, span, cyclic=cyclic)
res = {}
for d in range(rt.num_datasets):
    info = rt.dataset_info(d)
    a0, a1 = info["lo"][0], info["hi"][0]
    lo = own[0] if rank > 0 else a0
    hi = own[1] if rank + 1 < world else a1
    h = rt.host(d)
    res[f"rows{d}"] = np.array([lo, hi])
    res[f"stale{d}"] = np.array([int(info["stale"])])
    res[f"data{d}"] = np.ascontiguousarray(h[lo - a0:hi - a0])
res["ghost"] = np.array([ghost])
try:
    res["fieldsum"] = np.array([rt.fetch_reduction("fieldsum")])
except B.OocError:
    pass
dev = rt.device()
res["comm_bytes"] = np.array([dev["comm_bytes"]])
res["sweeps"] = np.array([dev.get("sweep_launches", 0)])
np.savez(out, **res)
rt.close()
