"""Child process of test_gpu_sweep.py::test_sweep_build_failure_falls_back: with
OOC_SWEEP_FAIL_BUILD set (read once per process) every row-sweep launch reports
OOC_ERR_UNSUPPORTED; the engine must fall back to the fused launches with the same
bits, and the measured timeline must bill each loop's bytes exactly once."""
import csv
import io
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_02125_b200 as B  # noqa: E402
from oracle import programs as P  # noqa: E402
from tests.helpers import compare, oracle_record, product_record  # noqa: E402

B.set_jit(2, 0)
bad = []
for app, nx, ny, iters, span in [("miniflow2d", 300, 256, 12, 0), ("rk3chain", 120, 100, 6, 3)]:
    prog = P.app_program(app, nx, ny, 0, iters=iters, span=span)
    want = oracle_record(prog, "reference")
    got = product_record(prog, "resident", timeline=True)
    rt = got.pop("_rt")
    want.pop("_rt", None)
    if compare(want, got, check_audit=False, check_totals=False):
        bad.append((app, "fields"))
    dev = rt.device()
    if dev["sweep_launches"] != 0:
        bad.append((app, "sweep launched", dev["sweep_launches"]))
    tl = [r for r in csv.DictReader(io.StringIO("\n".join(
        l for l in rt.timeline_csv().splitlines() if not l.startswith("#")))) if r["kind"] == "kernel"]
    kbytes = sum(int(r["bytes"]) for r in tl)
    if kbytes != rt.report()["total_bytes"]:
        bad.append((app, "timeline bytes", kbytes, rt.report()["total_bytes"]))
    print(app, "ok" if not bad else bad, flush=True)
print("BAD", bad)
sys.exit(1 if bad else 0)
