"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED reference.

    make -C oracle/ref && python tests/golden/make_golden.py

Needs oracle/_ref/libooc_ref.so (built from /root/reference/proj/src). Every
number written here comes from the reference library itself; the numpy
restatement (oracle/ooc_oracle.py) and the product are checked against these
files by tests/test_oracle_golden.py and tests/test_gpu_parity.py.

Fixture schema (all compact so the files stay small):
  random_programs.json: [{seed, kwargs, program_sha, runs: [...], plans: [...]}]
    run  = {executor, tiles, cyclic, error | {buffers, stale, reductions, audit_sha,
            totals, flush_log}}
    plan = {chain, tiles, sha, T, slot_bytes} for tiles in 1..4, plus budgeted choices
  apps.json: [{app, args, runs: [...]}] with the same run schema plus per-chain T.
Buffers are stored as oracle.ooc_oracle.checksum() digests; reductions as
float.hex() so comparisons are bitwise.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import programs as P  # noqa: E402
from oracle import refo  # noqa: E402
from oracle.ooc_oracle import checksum  # noqa: E402


def sha(obj) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True).encode()).hexdigest()[:24]


def reduction_names(prog):
    return sorted({op["kernel"]["reduction"]["name"] for op in prog["ops"]
                   if op["op"] == "loop" and "reduction" in op.get("kernel", {})})


def run_record(prog, executor, tiles=0, capacity=1 << 40, cyclic=False, extra=False,
               prefetch=False):
    pr = json.loads(json.dumps(prog))
    if cyclic:
        pr["ops"].insert(0, {"op": "cyclic", "on": True})
    ref = refo.RefRuntime(executor, tiles=tiles, capacity=capacity, record=True, prefetch=prefetch)
    rec = {"executor": executor, "tiles": tiles, "capacity": capacity, "cyclic": cyclic}
    if prefetch:
        rec["prefetch"] = True
    try:
        ref.load_program(pr)
    except refo.RefError as e:
        rec["error"] = e.kind
        return rec
    n = len(ref.datasets())
    rec["buffers"] = [checksum(ref.host(d)) for d in range(n)]
    rec["stale"] = [ref.stale(d) for d in range(n)]
    rec["reductions"] = {}
    for name in reduction_names(prog):
        try:
            rec["reductions"][name] = float.hex(ref.fetch_reduction(name))
        except refo.RefError:
            pass
    audit = ref.audit()
    rec["audit_sha"] = sha(audit)
    tot = ref.totals()
    rec["totals"] = [tot["uploaded"], tot["downloaded"], tot["d2d"], tot["metric_bytes"]]
    rec["flush_log"] = ref.flush_log()
    if extra and executor == "explicit":
        rec["chain_tiles"] = [ref.chain_plan(ci, tiles=tiles, budget=capacity)["T"]
                              if tiles == 0 else tiles for ci in range(ref.num_chains())]
    return rec


def plan_records(prog):
    ref = refo.RefRuntime("reference", record=True).load_program(prog)
    out = []
    for ci in range(ref.num_chains()):
        for T in (1, 2, 3, 4):
            jp = ref.chain_plan(ci, tiles=T)
            out.append({"chain": ci, "tiles": T, "sha": sha(jp), "T": jp["T"],
                        "slot_bytes": jp["slot_bytes"]})
            if T == 1:
                s1 = jp["slot_bytes"]
        for budget in (3 * s1, 2 * s1, (3 * s1) // 2, 4096):
            jb = ref.chain_plan(ci, tiles=0, budget=budget)
            if "error" in jb:
                out.append({"chain": ci, "budget": budget, "error": jb["error"].split(":")[0]})
            else:
                out.append({"chain": ci, "budget": budget, "sha": sha(jb), "T": jb["T"],
                            "slot_bytes": jb["slot_bytes"]})
    return out


RANDOM_SEEDS = range(120)
RANDOM_KW = dict(flushes=True)

APP_CASES = [
    ("heat2d", dict(nx=24, ny=20, iters=6)),
    ("heat2d", dict(nx=40, ny=33, iters=9, span=3)),
    ("miniflow2d", dict(nx=24, ny=20, iters=11)),
    ("miniflow2d", dict(nx=64, ny=64, iters=20)),
    ("rk3chain", dict(nx=24, ny=20, iters=6, span=2)),
    ("rk3chain", dict(nx=32, ny=32, iters=3, span=3)),
    ("miniflow3d", dict(nx=12, ny=10, nz=9, iters=11)),
    ("rk3chain3d", dict(nx=10, ny=9, nz=8, iters=3, span=3)),
]


def problem_bytes(prog):
    tot = 0
    for jd in prog["datasets"]:
        n = 1
        h = jd["halo"]
        for d, (lo, hi) in enumerate(zip(jd["core"]["lo"], jd["core"]["hi"])):
            n *= hi - lo + 2 * (h[d] if isinstance(h, list) else h)
        tot += n * jd["elem_bytes"]
    return tot


def main():
    cases = []
    for seed in RANDOM_SEEDS:
        prog = P.random_program(seed, **RANDOM_KW)
        runs = [run_record(prog, "reference")]
        for T in (1, 3):
            for cyc in (False, True):
                runs.append(run_record(prog, "explicit", tiles=T, cyclic=cyc))
        runs.append(run_record(prog, "explicit", tiles=3, prefetch=True))
        cases.append({"seed": seed, "kwargs": RANDOM_KW, "program_sha": sha(prog), "runs": runs,
                      "plans": plan_records(prog)})
    with open(os.path.join(HERE, "random_programs.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))

    apps = []
    for name, kw in APP_CASES:
        kw = dict(kw)
        prog = P.app_program(name, kw.pop("nx"), kw.pop("ny"), kw.pop("nz", 0), **kw)
        pb = problem_bytes(prog)
        runs = [run_record(prog, "reference"),
                run_record(prog, "explicit", tiles=3, extra=True),
                run_record(prog, "explicit", capacity=pb // 3, extra=True),
                run_record(prog, "explicit", capacity=pb // 3, cyclic=True, extra=True),
                run_record(prog, "explicit", tiles=3, prefetch=True)]
        apps.append({"app": name, "case": [name, dict(APP_CASES[len(apps)][1])],
                     "program_sha": sha(prog), "problem_bytes": pb, "runs": runs})
    with open(os.path.join(HERE, "apps.json"), "w") as f:
        json.dump(apps, f, separators=(",", ":"))

    # the reference's own run_app must agree with our program restatement of it
    for name, kw in APP_CASES:
        if name.endswith("3d"):
            continue
        ref = refo.RefRuntime("reference").run_app(name, kw["nx"], kw["ny"], kw["iters"],
                                                   kw.get("span", 0))
        prog = P.app_program(name, kw["nx"], kw["ny"], iters=kw["iters"], span=kw.get("span", 0))
        pr = refo.RefRuntime("reference").load_program(prog)
        for d in range(len(ref.datasets())):
            assert checksum(ref.host(d)) == checksum(pr.host(d)), (name, d)
    print("wrote", len(cases), "random cases and", len(apps), "app cases")


if __name__ == "__main__":
    main()
