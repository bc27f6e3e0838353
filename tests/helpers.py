"""Shared test helpers: run one program through the numpy oracle or the product and
produce a record in the golden-fixture schema (tests/golden/make_golden.py)."""
from __future__ import annotations

import hashlib
import json
import math

import numpy as np

from oracle import ooc_oracle as O

REL_TOL = 1e-12  # north_star: fp64 relative error on field summaries (reductions)


def sha(obj) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True).encode()).hexdigest()[:24]


def reduction_names(prog):
    return sorted({op["kernel"]["reduction"]["name"] for op in prog["ops"]
                   if op["op"] == "loop" and "reduction" in op.get("kernel", {})})


def with_cyclic(prog, cyclic):
    pr = json.loads(json.dumps(prog))
    if cyclic:
        pr["ops"].insert(0, {"op": "cyclic", "on": True})
    return pr


def oracle_record(prog, executor, tiles=0, capacity=1 << 40, cyclic=False, prefetch=False):
    rt = O.Runtime(executor, tiles=tiles, capacity=capacity, record=True, prefetch=prefetch)
    rec = {}
    try:
        O.load_program(rt, with_cyclic(prog, cyclic))
    except (O.ValidationError, O.StaleDataError, O.InfeasibleError, O.CapacityError) as e:
        rec["error"] = type(e).__name__
        return rec
    rec["buffers"] = [O.checksum(d.host) for d in rt.mesh]
    rec["stale"] = [d.host_stale for d in rt.mesh]
    rec["reductions"] = {n: float.hex(v) for n, v in rt.reductions.items()}
    rec["audit_sha"] = sha([list(r) for r in rt.audit])
    rec["totals"] = [rt.uploaded, rt.downloaded, rt.d2d, rt.metric_bytes]
    rec["flush_log"] = [list(f) for f in rt.flush_log]
    rec["_rt"] = rt
    return rec


def product_record(prog, executor, tiles=0, capacity=1 << 40, cyclic=False, **kw):
    import paper_1709_02125_b200 as B
    rt = B.Runtime(executor, tiles=tiles, capacity=capacity, record=True, **kw)
    rec = {}
    try:
        B.load_program(rt, with_cyclic(prog, cyclic))
    except (B.ValidationError, B.StaleDataError, B.InfeasibleError, B.CapacityError) as e:
        rec["error"] = type(e).__name__
        return rec
    rt.sync()
    n = rt.num_datasets
    rec["buffers"] = [O.checksum(rt.host(d)) for d in range(n)]
    rec["stale"] = [rt.dataset_info(d)["stale"] for d in range(n)]
    rec["reductions"] = {}
    for name in reduction_names(prog):
        try:
            rec["reductions"][name] = float.hex(rt.fetch_reduction(name))
        except B.OocError:
            pass
    audit = rt.audit()
    rec["audit_sha"] = sha(audit)
    rep = rt.report()
    rec["totals"] = [rep["uploaded"], rep["downloaded"], rep["d2d"], rep["total_bytes"]]
    rec["flush_log"] = rt.flush_log()
    rec["_rt"] = rt
    return rec


def close(a_hex, b_hex, tol=REL_TOL):
    a, b = float.fromhex(a_hex), float.fromhex(b_hex)
    if a == b or (math.isnan(a) and math.isnan(b)):
        return True
    return abs(a - b) <= tol * max(abs(a), abs(b))


def compare(want, got, *, exact_reductions=False, check_audit=True, check_totals=True):
    """Return a list of mismatch descriptions (empty = parity)."""
    bad = []
    if "error" in want or "error" in got:
        if want.get("error") != got.get("error"):
            bad.append(f"error {want.get('error')} != {got.get('error')}")
        return bad
    for i, (a, b) in enumerate(zip(want["buffers"], got["buffers"])):
        if a != b:
            bad.append(f"dataset {i} buffer differs")
    if want["stale"] != got["stale"]:
        bad.append(f"stale flags {want['stale']} != {got['stale']}")
    for name, v in want["reductions"].items():
        g = got["reductions"].get(name)
        if g is None:
            bad.append(f"reduction {name} missing")
        elif exact_reductions and g != v:
            bad.append(f"reduction {name} {v} != {g}")
        elif not close(v, g):
            bad.append(f"reduction {name} {float.fromhex(v)} vs {float.fromhex(g)} beyond {REL_TOL}")
    if check_audit and want["audit_sha"] != got["audit_sha"]:
        bad.append("audit rows differ")
    if check_totals and want["totals"][:3] != got["totals"][:3]:
        bad.append(f"transfer totals {want['totals'][:3]} != {got['totals'][:3]}")
    if want["totals"][3] != got["totals"][3]:
        bad.append(f"metric bytes {want['totals'][3]} != {got['totals'][3]}")
    if [list(x) for x in want["flush_log"]] != [list(x) for x in got["flush_log"]]:
        bad.append("flush log differs")
    return bad


def host_arrays(rt_product):
    return [np.array(rt_product.host(d)) for d in range(rt_product.num_datasets)]
