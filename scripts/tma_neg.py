import os, sys
sys.path.insert(0, os.getcwd())
import paper_1709_02125_b200 as B
from oracle import programs as P
from tests.helpers import compare, oracle_record, product_record
B.set_jit(2, 0)
case = sys.argv[1]
n = 300
p = P.Prog()
hx = 1 if case == "halo" else 0
p.declare("x", (0, 0), (n, 256), (hx, hx), "(+ 1.0 (* 0.001 i))")
p.declare("y", (-1, -1), (n + 1, 257), (0, 0), 0.0)
p.declare("z", (0, 0), (n, 256), (0, 0), 0.0)
if case in ("mixed", "halo"):
    p.loop((0, 0), (n, 256), [("x", P.POINT, P.R), ("z", P.POINT, P.W)], {1: P.mul(P.c(2.0), P.r(0))})
    p.loop((-1, -1), (n + 1, 257), [("y", P.POINT, P.W)], {0: P.c(3.0)})
else:
    p.loop((0, 0), (n, 256), [("x", P.POINT, P.R), ("z", P.POINT, P.W)], {1: P.mul(P.c(2.0), P.r(0))})
    p.loop((0, 0), (n, 256), [("y", P.POINT, P.W)], {0: P.c(3.0)})
p.finish()
prog = p.to_dict()
want = oracle_record(prog, "reference", tiles=1); want.pop("_rt", None)
got = product_record(prog, "reference", tiles=1); got.pop("_rt", None)
print(case, "diff", str(compare(want, got, check_audit=False, check_totals=False))[:300], flush=True)
