"""Pin the numpy restatement (oracle/ooc_oracle.py) to the reference.

Golden fixtures come from the unmodified reference library (tests/golden/make_golden.py);
the known-answer tests below are the reference's own (file:line cited)."""
import json

import numpy as np
import pytest

from oracle import ooc_oracle as O
from oracle import programs as P
from tests.helpers import compare, oracle_record, sha


def test_random_programs_match_reference_golden(golden_random):
    bad = []
    for case in golden_random:
        prog = P.random_program(case["seed"], **case["kwargs"])
        assert sha(prog) == case["program_sha"], "random program generator drifted"
        for want in case["runs"]:
            got = oracle_record(prog, want["executor"], want["tiles"], want["capacity"],
                                want["cyclic"], prefetch=want.get("prefetch", False))
            diff = compare(want, got, exact_reductions=True)
            if diff:
                bad.append((case["seed"], want["executor"], want["tiles"], want["cyclic"], diff))
    assert not bad, bad[:5]


def test_random_plans_match_reference_golden(golden_random):
    bad = []
    for case in golden_random[:60]:
        prog = P.random_program(case["seed"], **case["kwargs"])
        rt = O.load_program(O.Runtime("reference", record=True), prog)
        for p in case["plans"]:
            loops = rt.chain_log[p["chain"]]
            if "tiles" in p:
                plan = O.compute_tile_plan(rt.mesh, loops, p["tiles"])
                fp = O.compute_footprints(rt.mesh, loops, plan)
            else:
                try:
                    plan, fp = O.choose_tile_count(rt.mesh, loops, p["budget"])
                except O.InfeasibleError:
                    if p.get("error") != "InfeasibleError":
                        bad.append((case["seed"], p))
                    continue
            got = json.loads(json.dumps(O.plan_json(rt.mesh, plan, fp)))
            if sha(got) != p.get("sha"):
                bad.append((case["seed"], p))
    assert not bad, bad[:5]


def test_apps_match_reference_golden(golden_apps):
    bad = []
    for case in golden_apps:
        name, kw = case["case"]
        kw = dict(kw)
        prog = P.app_program(name, kw.pop("nx"), kw.pop("ny"), kw.pop("nz", 0), **kw)
        assert sha(prog) == case["program_sha"]
        for want in case["runs"]:
            got = oracle_record(prog, want["executor"], want["tiles"], want["capacity"],
                                want["cyclic"], prefetch=want.get("prefetch", False))
            diff = compare(want, got, exact_reductions=True)
            if diff:
                bad.append((name, want["executor"], want["tiles"], want["cyclic"], diff))
    assert not bad, bad


# ---------------------------------------------------------------- reference KATs


def _line3(halo=2):
    """proj/tests/test_tiler.cpp:26-48: fill a; b = a(+-1); c = b(+-1) on [0,12)."""
    rt = O.Runtime("reference", record=True)
    for n in "abc":
        rt.declare(n, O.Ext.make(1, (0,), (12,)), (halo,), 8, 0.0)
    pm1 = [(-1, 0, 0), (0, 0, 0), (1, 0, 0)]
    loops = [O.Loop(O.Ext.make(1, (0,), (12,)), [O.Arg(0, [(0, 0, 0)], O.WRITE)],
                    [(0, O.parse_prefix("1.0"))]),
             O.Loop(O.Ext.make(1, (0,), (12,)), [O.Arg(0, pm1, O.READ), O.Arg(1, [(0, 0, 0)], O.WRITE)],
                    [(1, O.parse_prefix("(r 0 0 0 0)"))]),
             O.Loop(O.Ext.make(1, (0,), (12,)), [O.Arg(1, pm1, O.READ), O.Arg(2, [(0, 0, 0)], O.WRITE)],
                    [(1, O.parse_prefix("(r 0 0 0 0)"))])]
    for i, l in enumerate(loops):
        O.validate_loop(rt.mesh, l)
        l.id = i
    return rt, loops


def test_kat_skew_accumulates():  # test_tiler.cpp:94-101
    rt, loops = _line3()
    plan = O.compute_tile_plan(rt.mesh, loops, 2)
    assert (plan.ends[2][0], plan.ends[1][0], plan.ends[0][0]) == (6, 7, 8)


def test_kat_golden_plan_json():  # test_tiler.cpp:340-367
    rt, loops = _line3(halo=1)
    plan = O.compute_tile_plan(rt.mesh, loops, 2)
    fp = O.compute_footprints(rt.mesh, loops, plan)
    assert fp.slot_bytes == 184
    assert plan.nominal_ends == [6, 12]
    fulls = [[pd.full[t].as_list() for pd in fp.per_dataset] for t in range(2)]
    assert fulls[0] == [[1, -1, 0, 0, 8, 1, 1], [1, -1, 0, 0, 7, 1, 1], [1, 0, 0, 0, 6, 1, 1]]
    assert fulls[1] == [[1, 6, 0, 0, 13, 1, 1], [1, 5, 0, 0, 13, 1, 1], [1, 6, 0, 0, 12, 1, 1]]
    assert [plan.subrange(j, 0).as_list()[1] for j in range(3)] == [0, 0, 0]
    assert [plan.subrange(j, 0).as_list()[4] for j in range(3)] == [8, 7, 6]


def test_kat_footprint_edges():  # test_tiler.cpp:247-273
    rt = O.Runtime()
    a = rt.declare("a", O.Ext.make(1, (0,), (12,)), (0,), 8, 0.0)
    b = rt.declare("b", O.Ext.make(1, (0,), (12,)), (0,), 8, 0.0)
    l1 = O.Loop(O.Ext.make(1, (0,), (12,)), [O.Arg(a, [(0, 0, 0)], O.WRITE)], [(0, ("const", 1.0))])
    l2 = O.Loop(O.Ext.make(1, (1,), (11,)),
                [O.Arg(a, [(-1, 0, 0), (0, 0, 0), (1, 0, 0)], O.READ), O.Arg(b, [(0, 0, 0)], O.WRITE)],
                [(1, ("read", 0, (0, 0, 0)))])
    for l in (l1, l2):
        O.validate_loop(rt.mesh, l)
    plan = O.compute_tile_plan(rt.mesh, [l1, l2], 2)
    pa = O.compute_footprints(rt.mesh, [l1, l2], plan).per_dataset[a]
    box = lambda lo, hi: [1, lo, 0, 0, hi, 1, 1]
    assert pa.full[0].as_list() == box(0, 7) and pa.full[1].as_list() == box(5, 12)
    assert pa.right_edge[0].as_list() == box(5, 7) and pa.left_fp[0].as_list() == box(0, 5)
    assert pa.left_edge[1].as_list() == box(5, 7) and pa.right_fp[1].as_list() == box(7, 12)
    assert pa.left_fp[1].as_list() == box(5, 12)
    assert pa.left_edge[0].empty() and pa.right_edge[1].empty()


def test_kat_kernels():  # test_mesh_core.cpp:66-117
    rt = O.Runtime()
    u = rt.declare("u", O.Ext.make(2, (0, 0), (8, 8)), (1, 1), 8, 1.0)
    w = rt.declare("w", O.Ext.make(2, (0, 0), (8, 8)), (1, 1), 8, 0.0)
    rt.enqueue_loop(O.Loop(O.Ext.make(2, (0, 0), (8, 8)),
                           [O.Arg(u, P.star(2), O.READ), O.Arg(w, [(0, 0, 0)], O.WRITE)],
                           [(1, O.parse_prefix(P.avg4(0)))]))
    assert np.all(rt.fetch_dataset(w)[1:9, 1:9] == 1.0)
    a = rt.declare("a", O.Ext.make(2, (0, 0), (4, 1)), (0, 0), 8, 41.0)
    rt.enqueue_loop(O.Loop(O.Ext.make(2, (0, 0), (4, 1)), [O.Arg(a, [(0, 0, 0)], O.RW)],
                           [(0, O.parse_prefix("(+ (r 0 0 0) 1.0)"))]))
    assert rt.fetch_dataset(a)[2, 0, 0] == 42.0


def test_kat_reduction_row_major_fold():  # test_mesh_core.cpp:94-117
    assert O.reduce_fold("SUM", 0.0, np.arange(4.0)) == 6.0
    # +0 / -0 ties keep the first extremum like std::min
    assert str(O.reduce_fold("MIN", float("inf"), np.array([0.0, -0.0]))) == "0.0"
    assert O.reduce_fold("MAX", -float("inf"), np.array([np.nan, 1.0])) == 1.0
