import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1709_02125_b200 as B
from oracle import programs as P
from tests.helpers import compare, oracle_record, product_record
B.set_jit(2, 0)
for app, nx, ny, nz, iters in [("heat2d", 200, 130, 0, 3), ("miniflow2d", 300, 256, 0, 4)]:
    prog = P.app_program(app, nx, ny, nz, iters=iters)
    want = oracle_record(prog, "explicit", tiles=1); want.pop("_rt", None)
    t0 = time.time()
    got = product_record(prog, "explicit", tiles=1); got.pop("_rt", None)
    print(app, "diff:", str(compare(want, got))[:500], time.time() - t0, flush=True)
print(B.jit_report())
