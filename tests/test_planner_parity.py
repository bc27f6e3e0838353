"""Product planner + lazy runtime (libooc.so, plan_only executor: no device needed)
against the reference: plans must match bit-exactly (north_star)."""
import json
import os

import numpy as np
import pytest

import paper_1709_02125_b200 as B
from oracle import programs as P
from oracle import ooc_oracle as O
from tests.helpers import sha


def plan_only(prog, **kw):
    return B.load_program(B.Runtime("plan_only", record=True, tiles=1, **kw), prog)


def test_random_plans_bit_exact(golden_random):
    bad = []
    for case in golden_random:
        prog = P.random_program(case["seed"], **case["kwargs"])
        rt = plan_only(prog)
        for p in case["plans"]:
            try:
                if "tiles" in p:
                    got = rt.chain_plan(p["chain"], tiles=p["tiles"])
                else:
                    got = rt.chain_plan(p["chain"], budget=p["budget"])
            except B.InfeasibleError:
                if p.get("error") != "InfeasibleError":
                    bad.append((case["seed"], p))
                continue
            if sha(got) != p.get("sha"):
                bad.append((case["seed"], p))
    assert not bad, bad[:5]


def test_flush_logs_match(golden_random):
    for case in golden_random:
        prog = P.random_program(case["seed"], **case["kwargs"])
        rt = plan_only(prog)
        assert rt.flush_log() == case["runs"][0]["flush_log"]


@pytest.mark.parametrize("app,kw", [
    ("heat2d", dict(nx=40, ny=33, iters=9, span=3)),
    ("miniflow2d", dict(nx=64, ny=64, iters=20)),
    ("rk3chain", dict(nx=32, ny=32, iters=3, span=3)),
    ("miniflow3d", dict(nx=12, ny=10, nz=9, iters=11)),
    ("rk3chain3d", dict(nx=10, ny=9, nz=8, iters=3, span=3)),
])
def test_native_apps_equal_program_restatement(app, kw):
    """The product's C++ apps build the same chains and fills as the chain-file
    programs the reference runs (oracle/programs.py)."""
    prog = P.app_program(app, kw["nx"], kw["ny"], kw.get("nz", 0), iters=kw["iters"],
                         span=kw.get("span", 0))
    a = plan_only(prog)
    b = B.Runtime("plan_only", record=True, tiles=1)
    b.run_app(app, kw["nx"], kw["ny"], kw.get("nz", 0), kw["iters"], kw.get("span", 0))
    assert a.flush_log() == b.flush_log()
    for ci in range(a.num_chains()):
        for T in (1, 2, 5):
            assert a.chain_plan(ci, tiles=T) == b.chain_plan(ci, tiles=T)
    for d in range(a.num_datasets):
        assert np.array_equal(a.host(d).view(np.uint64), b.host(d).view(np.uint64))
    # and the fills equal the numpy restatement's (bit-exact)
    o = O.load_program(O.Runtime(), {"datasets": prog["datasets"], "ops": []})
    for d in range(a.num_datasets):
        assert np.array_equal(a.host(d).view(np.uint64), o.mesh[d].host.view(np.uint64))


def test_problem_bytes():
    # miniflow2d 960^2: 4 halo-2 fields + 6 temporaries (74.2 MB)
    assert B.problem_bytes("miniflow2d", 960, 960) == (4 * 964 * 964 + 6 * 962 * 962) * 8


# ---------------------------------------------------------------- reference KATs


def _line3_prog(halo=2):
    p = P.Prog()
    for n in "abc":
        p.declare(n, (0,), (12,), (halo,), 0.0)
    pm1 = P.line(0)
    p.loop((0,), (12,), [("a", P.POINT, P.W)], {0: "1.0"})
    p.loop((0,), (12,), [("a", pm1, P.R), ("b", P.POINT, P.W)], {1: "(r 0 0 0 0)"})
    p.loop((0,), (12,), [("b", pm1, P.R), ("c", P.POINT, P.W)], {1: "(r 0 0 0 0)"})
    p.finish()
    return p.to_dict()


def test_kat_golden_plan_dump_json():  # proj/tests/test_tiler.cpp:340-367
    rt = plan_only(_line3_prog(halo=1))
    got = rt.chain_plan(0, tiles=2, dump=True)
    want = {
        "tiled_dim": 0, "tiles": 2, "slot_bytes": 184, "nominal_ends": [6, 12],
        "tiles_detail": [
            {"tile": 0,
             "loops": [{"loop": 0, "empty": False, "range": {"lo": [0], "hi": [8]}},
                       {"loop": 1, "empty": False, "range": {"lo": [0], "hi": [7]}},
                       {"loop": 2, "empty": False, "range": {"lo": [0], "hi": [6]}}],
             "datasets": [
                 {"dataset": "a", "full": {"lo": [-1], "hi": [8]}, "bytes": 72, "modified": True},
                 {"dataset": "b", "full": {"lo": [-1], "hi": [7]}, "bytes": 64, "modified": True},
                 {"dataset": "c", "full": {"lo": [0], "hi": [6]}, "bytes": 48, "modified": True}]},
            {"tile": 1,
             "loops": [{"loop": 0, "empty": False, "range": {"lo": [8], "hi": [12]}},
                       {"loop": 1, "empty": False, "range": {"lo": [7], "hi": [12]}},
                       {"loop": 2, "empty": False, "range": {"lo": [6], "hi": [12]}}],
             "datasets": [
                 {"dataset": "a", "full": {"lo": [6], "hi": [13]}, "bytes": 56, "modified": True},
                 {"dataset": "b", "full": {"lo": [5], "hi": [13]}, "bytes": 64, "modified": True},
                 {"dataset": "c", "full": {"lo": [6], "hi": [12]}, "bytes": 48, "modified": True}]}]}
    assert got == want
    text = rt.chain_plan_text(0, 2)
    assert "tile 0" in text and "loop 0 range [0,8)" in text


def test_kat_skew_and_oracle():  # test_tiler.cpp:94-125
    rt = plan_only(_line3_prog())
    plan = rt.chain_plan(0, tiles=2)
    assert [plan["ends"][j][0] for j in (2, 1, 0)] == [6, 7, 8]
    assert rt.chain_oracle(0, 2)["ok"]


def test_kat_tile_count_reduced_with_warning():  # test_tiler.cpp:136-147
    p = P.Prog()
    p.declare("a", (0,), (4,), (0,), 0.0)
    p.loop((0,), (4,), [("a", P.POINT, P.W)], {0: "1.0"})
    p.finish()
    plan = plan_only(p.to_dict()).chain_plan(0, tiles=9)
    assert plan["T"] == 4 and plan["warnings"] == 1


def test_kat_choose_tile_count():  # test_tiler.cpp:294-313
    rt = plan_only(_line3_prog())
    problem = 3 * 16 * 8
    assert rt.chain_plan(0, budget=3 * problem)["T"] == 1
    halves = rt.chain_plan(0, budget=3 * problem * 3 // 4)
    assert halves["T"] > 1 and 3 * halves["slot_bytes"] <= 3 * problem * 3 // 4
    with pytest.raises(B.InfeasibleError):
        rt.chain_plan(0, budget=8)


# ---------------------------------------------------------------- lazy queue semantics


def test_lazy_queue_and_reduction_flush():  # test_lazy_queue.cpp:28-56, 114-128
    rt = B.Runtime("plan_only", record=True)
    d = rt.declare("d", (0,), (8,), (0,), 1.0)
    for _ in range(3):
        rt.enqueue_loop((0,), (8,), [(d, B.POINT, B.READ_WRITE)], {0: "(+ (r 0 0 0 0) 1.0)"})
    assert rt.num_chains() == 0
    rt.enqueue_loop((0,), (8,), [(d, B.POINT, B.READ)], None, ("SUM", "(r 0 0 0 0)", "total"))
    assert rt.flush_log() == [[0, "REDUCTION_FETCH", 4]]
    rt.finish()
    assert rt.flush_log() == [[0, "REDUCTION_FETCH", 4]]  # nothing pending: no extra chain


def test_fetch_without_pending_returns_fill():  # test_lazy_queue.cpp:58-64
    rt = B.Runtime("plan_only")
    d = rt.declare("d", (0,), (4,), (0,), 7.0)
    assert np.all(rt.fetch_dataset(d) == 7.0)


@pytest.mark.parametrize("bad", [
    dict(lo=(0,), hi=(0,), args="w", msg="empty iteration range"),
    dict(lo=(0,), hi=(9,), args="w", msg="exceeds the core"),
    dict(lo=(0,), hi=(8,), args="wide", msg="single zero-offset"),
    dict(lo=(0,), hi=(8,), args="dup", msg="appears in another argument"),
    dict(lo=(0,), hi=(8,), args="noexpr", msg="never writes"),
])
def test_validation_errors(bad):  # proj/src/loop.cpp:32-105
    rt = B.Runtime("plan_only")
    d = rt.declare("d", (0,), (8,), (1,), 0.0)
    e = rt.declare("e", (0,), (8,), (1,), 0.0)
    args = {"w": ([(d, B.POINT, B.WRITE)], {0: "1.0"}),
            "wide": ([(d, B.line(0), B.WRITE)], {0: "1.0"}),
            "dup": ([(d, B.POINT, B.WRITE), (d, B.POINT, B.READ)], {0: "1.0"}),
            "noexpr": ([(d, B.POINT, B.WRITE), (e, B.POINT, B.READ)], {})}[bad["args"]]
    with pytest.raises(B.ValidationError, match=bad["msg"]):
        rt.enqueue_loop(bad["lo"], bad["hi"], *args)


def test_out_of_scope_executors_rejected():
    import ctypes
    from paper_1709_02125_b200 import _native
    o = _native.Options()
    _native.lib().ooc_rt_default_options(ctypes.byref(o))
    o.executor = 1  # tiled_cache: KNL cost model, not part of the B200 build
    h = ctypes.c_void_p()
    assert _native.lib().ooc_rt_create(ctypes.byref(o), ctypes.byref(h)) == -1


@pytest.mark.parametrize("app,kw", [("miniflow2d", dict(nx=64, ny=48, iters=12)),
                                    ("rk3chain3d", dict(nx=10, ny=9, nz=8, iters=3, span=3))])
def test_specialised_kernels_compile_for_sm100a(app, kw):
    """The NVRTC-instantiated par_loop kernels of every fused group build for sm_100a."""
    if not B.jit_status() in ("ok", "libcuda.so.1 (driver) not available"):
        pytest.skip("NVRTC unavailable: " + B.jit_status())
    rt = B.Runtime("plan_only", record=True, tiles=1)
    rt.run_app(app, kw["nx"], kw["ny"], kw.get("nz", 0), kw["iters"], kw.get("span", 0))
    groups = rt.chain_jit_check(rt.num_chains() - 1, fuse=True)
    assert groups and all(g["ok"] for g in groups), [g.get("log", "")[:500] for g in groups if not g["ok"]]
    assert max(g["loops"] for g in groups) > 1  # fusion happened


def test_report_csv_schemas_match_reference():
    """proj/src/metrics.cpp:46-79 / command.cpp:160-168 headers; one loops row per loop."""
    prog = P.app_program("heat2d", 32, 32, 0, iters=2)
    rt = plan_only(prog)
    rep = rt.report_csv("heat2d", "32x32", 2).splitlines()
    assert rep[0] == "#oocstencil-report-v1"
    assert rep[1] == ("app,size,iters,mode,tiles,capacity,average_bandwidth,total_bytes,"
                      "total_time,makespan,uploaded,downloaded,d2d,efficiency,hit_rate,faults,error")
    assert rep[2].startswith("heat2d,32x32,2,plan_only,1,")
    loops = rt.loops_csv().splitlines()
    assert loops[:2] == ["#oocstencil-report-v1", "loop,points,bytes,time,bandwidth"]
    assert [l.split(",")[0] for l in loops[2:]] == ["0", "1"]
    assert rt.audit_csv() == "dataset,tile,uploaded,downloaded,d2d\n"
    assert rt.timeline_csv() == "command_id,kind,queue,bytes,issue,start,end\n"


def test_fusion_plan_miniflow2d():
    """Least-traffic legal partition: per iteration [L1-L6] (stencil reads of rho/e/v),
    [L7-L13], [L14]; with row recompute [L7-L14] (L14's row-offset read of t3 is
    re-evaluated in-thread from L10/L11). The fieldsum reduction runs alone."""
    rt = B.Runtime("plan_only", record=True, tiles=1)
    rt.run_app("miniflow2d", 64, 48, 0, 22)
    c = rt.num_chains() - 2  # iterations 10..19: a full 10-iteration chain
    assert [g["loops"] for g in rt.chain_jit_check(c, fuse=False)][:3] == [1, 1, 1]
    if B.jit_status() not in ("ok", "libcuda.so.1 (driver) not available"):
        pytest.skip("NVRTC unavailable")
    try:
        for on, want in ((False, [6, 7, 1] * 10 + [1]), (True, [6, 8] * 10 + [1])):
            B.set_row_recompute(on)
            got = rt.chain_jit_check(c, fuse=True)
            assert [g["loops"] for g in got] == want
            assert all(g["ok"] for g in got)
    finally:
        B.set_row_recompute(os.environ.get("OOC_ROW_RECOMPUTE", "1") != "0")


@pytest.mark.parametrize("shape", ["t16x64", "t8x64", "t4x64"])
def test_tma_template_compiles_for_sm100a(shape):
    """The shared-memory/TMA kernel template builds for sm_100a for every fused group of
    the 2-D and 3-D apps (child process: OOC_JIT_SHAPE is read once per process)."""
    import subprocess
    import sys
    if B.jit_status() not in ("ok", "libcuda.so.1 (driver) not available"):
        pytest.skip("NVRTC unavailable")
    code = (
        "import paper_1709_02125_b200 as B\n"
        "for app, nz, span in (('miniflow2d', 0, 0), ('miniflow3d', 24, 0), ('rk3chain3d', 20, 3)):\n"
        "    rt = B.Runtime('plan_only', record=True, tiles=1)\n"
        "    rt.run_app(app, 40, 36, nz, 6, span)\n"
        "    g = rt.chain_jit_check(rt.num_chains() - 1, fuse=True)\n"
        "    bad = [x.get('log', '')[:800] for x in g if not x['ok'] and 'capacity' not in x.get('log', '')]\n"
        "    assert g and not bad, (app, bad)  # groups over the smem budget fall back to registers\n"
        "    assert any('<<TMA>>' in x.get('log', '') for x in g), app\n")
    env = dict(__import__("os").environ, OOC_JIT_SHAPE=shape, OOC_JIT_DUMP="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__)), timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
