"""Child process of test_gpu_parity.py::test_forced_tile_shapes: with OOC_JIT_SHAPE set
in the environment (read once per process), every specialised launch uses that one tile
shape; compare medium apps and random programs with the oracle. Exit 0 = parity."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_02125_b200 as B  # noqa: E402
from oracle import programs as P  # noqa: E402
from tests.helpers import compare, oracle_record, product_record  # noqa: E402

B.set_jit(2, 0)
if os.environ.get("OOC_ROW_RECOMPUTE") == "1":
    B.set_row_recompute(True)
bad = []
for app, nx, ny, nz, iters, span in [("miniflow2d", 300, 256, 0, 12, 0), ("miniflow3d", 40, 36, 30, 10, 0),
                                     ("rk3chain3d", 30, 28, 26, 6, 3), ("heat2d", 200, 130, 0, 7, 0)]:
    prog = P.app_program(app, nx, ny, nz, iters=iters, span=span)
    pb = B.problem_bytes(app, nx, ny, nz, span)
    for kw in (dict(capacity=pb // 2), dict(tiles=1)):
        want = oracle_record(prog, "explicit", **kw)
        got = product_record(prog, "explicit", **kw)
        want.pop("_rt", None)
        got.pop("_rt", None)
        d = compare(want, got)
        print(app, kw, "ok" if not d else "DIFF", flush=True)
        if d:
            bad.append((app, kw, str(d)[:300]))
for seed in range(20):
    prog = P.random_program(seed, flushes=True)
    want = oracle_record(prog, "explicit", tiles=3)
    got = product_record(prog, "explicit", tiles=3)
    want.pop("_rt", None)
    got.pop("_rt", None)
    if compare(want, got):
        bad.append(("random", seed))
print("launches", B.Runtime("resident").device()["jit_launches"], "report", B.jit_report()[:2])
print("BAD", bad)
sys.exit(1 if bad else 0)
