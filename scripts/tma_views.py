import os, sys
sys.path.insert(0, os.getcwd())
import paper_1709_02125_b200 as B
from oracle import programs as P
from tests.helpers import compare, oracle_record, product_record
B.set_jit(2, 0)
k = int(sys.argv[1])
p = P.Prog()
names = [f"d{i}" for i in range(k)]
for i, nm in enumerate(names):
    p.declare(nm, (0, 0), (300, 256), (1, 1), f"(+ {i}.0 (* 0.001 i))")
p.declare("out", (0, 0), (300, 256), (1, 1), 0.0)
expr = P.r(0)
for i in range(1, k):
    expr = P.add(expr, P.r(i))
p.loop((0, 0), (300, 256), [(nm, P.POINT, P.R) for nm in names] + [("out", P.POINT, P.W)], {k: expr})
p.finish()
prog = p.to_dict()
want = oracle_record(prog, "explicit", tiles=1); want.pop("_rt", None)
got = product_record(prog, "explicit", tiles=1); got.pop("_rt", None)
print("views", k, "diff", str(compare(want, got))[:200], flush=True)
