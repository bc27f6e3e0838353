"""Parity probe: one app through the resident executor vs the oracle (env selects the
sweep variant). python scripts/sweep_rk_child.py app nx ny iters span"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1709_02125_b200 as B  # noqa: E402
from oracle import ooc_oracle as O  # noqa: E402
from oracle import programs as P  # noqa: E402

app, nx, ny, iters, span = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
B.set_jit(2, 0)
prog = P.app_program(app, nx, ny, 0, iters=iters, span=span)
rt = B.load_program(B.Runtime("resident", record=True), prog)
ref = O.load_program(O.Runtime("reference"), prog)
bad = []
for d in range(rt.num_datasets):
    got = np.asarray(rt.fetch_dataset(d))
    want = ref.mesh[d].host
    if not np.array_equal(got.view(np.uint64), want.view(np.uint64)):
        idx = np.argwhere(got.view(np.uint64) != want.view(np.uint64))
        bad.append((d, len(idx), idx[:3].tolist(), idx[-3:].tolist()))
print({k: os.environ.get(k) for k in ("OOC_SWEEP_FWD", "OOC_SWEEP_SMEM")}, "sweeps", rt.device()["sweep_launches"],
      "BAD" if bad else "ok", bad)
