"""Child process of test_gpu_sweep.py::test_sweep_variants (OOC_SWEEP_K / _P / _SMEM
are read once per process): resident apps and random programs vs the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_02125_b200 as B  # noqa: E402
from oracle import programs as P  # noqa: E402
from tests.helpers import compare, oracle_record, product_record  # noqa: E402

B.set_jit(2, 0)
bad, swept = [], 0
cases = [("miniflow2d", 300, 256, 12, 0), ("miniflow2d", 131, 77, 21, 0), ("heat2d", 200, 130, 7, 0),
         ("rk3chain", 120, 100, 6, 3)]
for app, nx, ny, iters, span in cases:
    prog = P.app_program(app, nx, ny, 0, iters=iters, span=span)
    want = oracle_record(prog, "reference")
    got = product_record(prog, "resident")
    rt = got.pop("_rt")
    swept += rt.device()["sweep_launches"]
    want.pop("_rt", None)
    d = compare(want, got, check_audit=False, check_totals=False)
    print(app, nx, ny, "ok" if not d else "DIFF", flush=True)
    if d:
        bad.append((app, str(d)[:300]))
for seed in range(30):
    prog = P.random_program(seed, flushes=True)
    want = oracle_record(prog, "reference")
    got = product_record(prog, "resident")
    rt = got.pop("_rt")
    swept += rt.device()["sweep_launches"]
    want.pop("_rt", None)
    if compare(want, got, check_audit=False, check_totals=False):
        bad.append(("random", seed))
for seed in range(12):  # larger meshes: interior strips take the fast steps
    prog = P.random_program(seed, max_loops=12, min_size=300, max_size=700, allow_3d=False, flushes=True)
    want = oracle_record(prog, "reference")
    got = product_record(prog, "resident")
    rt = got.pop("_rt")
    swept += rt.device()["sweep_launches"]
    want.pop("_rt", None)
    if compare(want, got, check_audit=False, check_totals=False):
        bad.append(("large random", seed))
print("sweeps", swept, "BAD", bad)
sys.exit(1 if bad or swept == 0 else 0)
