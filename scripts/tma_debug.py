import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_1709_02125_b200 as B
from oracle import programs as P
from tests.helpers import compare, oracle_record, product_record
B.set_jit(2, 0)
mode = sys.argv[1]
if mode == "unfused":
    prog = P.app_program("miniflow2d", 300, 256, 0, iters=2)
    want = oracle_record(prog, "explicit", tiles=1); want.pop("_rt", None)
    got = product_record(prog, "explicit", tiles=1, fuse=False); got.pop("_rt", None)
    print("unfused diff", str(compare(want, got))[:300], flush=True)
elif mode == "random":
    for seed in range(int(sys.argv[2]), int(sys.argv[3])):
        prog = P.random_program(seed, flushes=True)
        want = oracle_record(prog, "explicit", tiles=1); want.pop("_rt", None)
        try:
            got = product_record(prog, "explicit", tiles=1, fuse=False); got.pop("_rt", None)
            print(seed, "diff", str(compare(want, got))[:200], flush=True)
        except Exception as e:
            print(seed, "ERR", str(e)[:200], flush=True)
            break
