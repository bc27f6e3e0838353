"""Sweep-kernel fuzzing against the numpy oracle (GPU; not part of the test suite):
random 2-D chains on 300-700 point meshes and random 3-D chains, resident, every field
bitwise and every reduction within 1e-12. Environment knobs (OOC_SWEEP_RC, ...) select
the schedule under test.

    python scripts/fuzz_sweeps.py [first_seed] [count]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1709_02125_b200 as B  # noqa: E402
from oracle import programs as P  # noqa: E402
from tests.helpers import compare, oracle_record, product_record  # noqa: E402

B.set_jit(2, 0)
first = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
count = int(sys.argv[2]) if len(sys.argv) > 2 else 60
bad, swept, n = [], 0, 0
for seed in range(first, first + count):
    for kind in ("2d", "3d"):
        if kind == "2d":
            prog = P.random_program(seed, max_loops=14, min_size=300, max_size=700, allow_3d=False, flushes=True)
        else:
            prog = P.random_program(seed, force_ndim=3, min_size=20, max_size=48, max_3d=48, flushes=True)
        want = oracle_record(prog, "reference")
        got = product_record(prog, "resident")
        rt = got.pop("_rt", None)
        want.pop("_rt", None)
        if rt is not None:
            swept += rt.device()["sweep_launches"]
        d = compare(want, got, check_audit=False, check_totals=False)
        n += 1
        if d:
            bad.append((seed, kind, str(d)[:200]))
            print("MISMATCH", seed, kind, d, flush=True)
env = {k: v for k, v in os.environ.items() if k.startswith("OOC_")}
print({"env": env, "programs": n, "sweep_launches": swept, "mismatches": len(bad)}, flush=True)
sys.exit(1 if bad else 0)
