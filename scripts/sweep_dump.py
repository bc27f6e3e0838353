"""Dump the generated row-sweep kernel of one run of a miniflow2d chain (source +
ptxas report) and its plan: python scripts/sweep_dump.py [run] [out.cu]."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("OOC_JIT_VERBOSE", "1")
out = sys.argv[2] if len(sys.argv) > 2 else "/tmp/sweep_k.cu"
os.environ["OOC_SWEEP_DUMP"] = out
import paper_1709_02125_b200 as B  # noqa: E402
from oracle import programs as P  # noqa: E402

B.set_jit(2, 0)
rt = B.load_program(B.Runtime("plan_only", record=True, tiles=1), P.app_program("miniflow2d", 64, 64, iters=10))
runs = rt.chain_sweep_check(rt.num_chains() - 1, compile=False)
k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
print([(g["first"], g["loops"], g["plan"]["smem"], g["dead"]) for g in runs])
g = rt.chain_sweep_check(rt.num_chains() - 1, compile=True)[k]
print(json.dumps(g["plan"])[:400])
print(open(out).read().split("/*")[-1][-400:])
