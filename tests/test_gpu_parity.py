"""GPU parity: the product's CUDA path (libooc.so -> liboocdev.so, sm_100a) against
the reference's golden fixtures and the numpy oracle. Fields bit-exact; reductions
within 1e-12 relative (north_star); audit bytes / stale flags / flush logs exact."""
import json

import numpy as np
import pytest

import paper_1709_02125_b200 as B
from oracle import ooc_oracle as O
from oracle import programs as P
from tests.helpers import REL_TOL, compare, oracle_record, product_record

pytestmark = pytest.mark.gpu

EXEC_OF = {"reference": "reference", "explicit": "explicit"}


def test_random_programs_vs_reference_golden(golden_random):
    bad = []
    for case in golden_random:
        prog = P.random_program(case["seed"], **case["kwargs"])
        for want in case["runs"]:
            got = product_record(prog, EXEC_OF[want["executor"]], want["tiles"], want["capacity"],
                                 want["cyclic"], prefetch=want.get("prefetch", False))
            got.pop("_rt", None)
            # the reference executor moves no bytes; only explicit runs carry an audit
            diff = compare(want, got, check_audit=want["executor"] == "explicit",
                           check_totals=want["executor"] == "explicit")
            if diff:
                bad.append((case["seed"], want["executor"], want["tiles"], want["cyclic"], diff))
    assert not bad, bad[:5]


def test_apps_vs_reference_golden(golden_apps):
    bad = []
    for case in golden_apps:
        name, kw = case["case"]
        kw = dict(kw)
        prog = P.app_program(name, kw.pop("nx"), kw.pop("ny"), kw.pop("nz", 0), **kw)
        for want in case["runs"]:
            got = product_record(prog, EXEC_OF[want["executor"]], want["tiles"], want["capacity"],
                                 want["cyclic"], prefetch=want.get("prefetch", False))
            got.pop("_rt", None)
            diff = compare(want, got, check_audit=want["executor"] == "explicit",
                           check_totals=want["executor"] == "explicit")
            if diff:
                bad.append((name, want["executor"], want["tiles"], want["cyclic"], diff))
    assert not bad, bad


def test_exact_reductions_vs_reference_golden(golden_random, golden_apps):
    """Exact mode (ooc_rt_set_exact_reductions): every reduction bit-equal to the
    reference's sequential fold, resident and streamed, across tile counts."""
    bad = []
    cases = [(P.random_program(c["seed"], **c["kwargs"]), c["runs"]) for c in golden_random]
    for c in golden_apps:
        name, kw = c["case"]
        kw = dict(kw)
        cases.append((P.app_program(name, kw.pop("nx"), kw.pop("ny"), kw.pop("nz", 0), **kw), c["runs"]))
    nred = 0
    for prog, runs in cases:
        for want in runs:
            got = product_record(prog, EXEC_OF[want["executor"]], want["tiles"], want["capacity"],
                                 want["cyclic"], prefetch=want.get("prefetch", False),
                                 exact_reductions=True)
            got.pop("_rt", None)
            nred += len(want.get("reductions", {}))
            diff = compare(want, got, exact_reductions=True, check_audit=want["executor"] == "explicit",
                           check_totals=want["executor"] == "explicit")
            if diff:
                bad.append((want["executor"], want["tiles"], want["cyclic"], diff))
    assert not bad, bad[:5]
    assert nred > 50


@pytest.mark.parametrize("fill", [1, 2])
def test_arena_initialisation_is_unobservable(fill):
    """Zero (reference) or NaN-poisoned arenas give identical results: no kernel
    ever reads a slot byte that was neither uploaded, carried nor written."""
    for seed in range(40):
        prog = P.random_program(seed, flushes=True)
        want = oracle_record(prog, "explicit", tiles=3)
        got = product_record(prog, "explicit", tiles=3, arena_fill=fill)
        want.pop("_rt", None)
        got.pop("_rt", None)
        assert not compare(want, got), seed


@pytest.mark.parametrize("T", [2, 4, 5, 8])
def test_more_tile_counts_vs_oracle(T):
    for seed in range(200, 240):
        prog = P.random_program(seed, flushes=True)
        for cyc in (False, True):
            want = oracle_record(prog, "explicit", tiles=T, cyclic=cyc)
            got = product_record(prog, "explicit", tiles=T, cyclic=cyc)
            want.pop("_rt", None)
            got.pop("_rt", None)
            assert not compare(want, got), (seed, T, cyc)


@pytest.mark.parametrize("app,nx,ny,nz,iters,span", [
    ("miniflow2d", 256, 200, 0, 20, 0),
    ("rk3chain", 200, 256, 0, 6, 3),
    ("heat2d", 300, 256, 0, 12, 4),
    ("miniflow3d", 40, 36, 30, 10, 0),
    ("rk3chain3d", 32, 30, 28, 3, 3),
])
@pytest.mark.parametrize("mode", ["resident", "explicit3", "explicit_cyclic", "l2tiled", "unfused"])
def test_apps_medium_vs_oracle(app, nx, ny, nz, iters, span, mode):
    prog = P.app_program(app, nx, ny, nz, iters=iters, span=span, cyclic=(mode == "explicit_cyclic"))
    pb = B.problem_bytes(app, nx, ny, nz, span)
    if mode == "resident":
        want = oracle_record(prog, "reference")
        got = product_record(prog, "resident")
        kw = dict(check_audit=False, check_totals=False)
    elif mode == "l2tiled":
        want = oracle_record(prog, "reference")
        got = product_record(prog, "resident", tiles=3)
        kw = dict(check_audit=False, check_totals=False)
    elif mode == "unfused":
        want = oracle_record(prog, "explicit", capacity=pb // 2)
        got = product_record(prog, "explicit", capacity=pb // 2, fuse=False)
        kw = {}
    else:
        want = oracle_record(prog, "explicit", capacity=pb // 2)
        got = product_record(prog, "explicit", capacity=pb // 2)
        kw = {}
    want.pop("_rt", None)
    got.pop("_rt", None)
    diff = compare(want, got, **kw)
    assert not diff, diff


def test_native_app_equals_program_on_gpu():
    """run_app through the C++ API == the chain-file program (fields bit-exact)."""
    prog = P.app_program("miniflow2d", 128, 96, iters=12)
    cap = B.problem_bytes("miniflow2d", 128, 96) // 2
    a = B.load_program(B.Runtime("explicit", capacity=cap), prog)
    b = B.Runtime("explicit", capacity=cap)
    b.run_app("miniflow2d", 128, 96, 0, 12)
    for d in range(a.num_datasets):
        assert np.array_equal(a.host(d).view(np.uint64), b.host(d).view(np.uint64))
    assert a.fetch_reduction("fieldsum") == b.fetch_reduction("fieldsum")


def test_l2_budget_tiling_miniflow():
    prog = P.app_program("miniflow2d", 256, 200, iters=20)
    pb = B.problem_bytes("miniflow2d", 256, 200)
    want = oracle_record(prog, "reference")
    got = product_record(prog, "resident", resident_budget=pb // 4)
    want.pop("_rt", None)
    got.pop("_rt", None)
    assert not compare(want, got, check_audit=False, check_totals=False)


def test_fieldsum_large_within_tolerance():
    """Parallel reduction tree vs the reference's sequential row-major fold."""
    n = 960
    prog = P.app_program("miniflow2d", n, n, iters=10)
    want = oracle_record(prog, "reference")
    got = product_record(prog, "resident")
    a = float.fromhex(want["reductions"]["fieldsum"])
    b = float.fromhex(got["reductions"]["fieldsum"])
    assert abs(a - b) <= REL_TOL * abs(a)
    assert want["buffers"] == got["buffers"]


def test_stale_fetch_raises_and_guard():  # test_lazy_queue.cpp:130-201
    rt = B.Runtime("explicit", tiles=2, capacity=1 << 40)
    rt.set_cyclic_flag(True)
    tmp = rt.declare("tmp", (0,), (16,), (0,), 0.0)
    out = rt.declare("out", (0,), (16,), (0,), 0.0)
    rt.enqueue_loop((0,), (16,), [(tmp, B.POINT, B.WRITE)], {0: "5.0"})
    rt.flush()
    assert rt.dataset_info(tmp)["stale"]
    with pytest.raises(B.StaleDataError):
        rt.fetch_dataset(tmp)
    rt.enqueue_loop((0,), (16,), [(tmp, B.POINT, B.READ), (out, B.POINT, B.WRITE)], {1: "(r 0 0)"})
    with pytest.raises(B.StaleDataError):
        rt.flush()


def test_capacity_error():  # test_device_sim.cpp:510-515
    rt = B.Runtime("explicit", tiles=2, capacity=64)
    a = rt.declare("a", (0,), (12,), (1,), 0.0)
    rt.enqueue_loop((0,), (12,), [(a, B.POINT, B.WRITE)], {0: "1.0"})
    with pytest.raises(B.CapacityError):
        rt.flush()


def test_edge_carry_known_answer():  # test_device_sim.cpp:158-167 (b[6] == 13)
    rt = B.Runtime("explicit", tiles=2, capacity=1 << 40)
    a = rt.declare("a", (0,), (12,), (1,), 0.0)
    b = rt.declare("b", (0,), (12,), (1,), 0.0)
    rt.enqueue_loop((0,), (12,), [(a, B.POINT, B.WRITE)], {0: "(+ 10.0 (* 3.0 1.0))"})
    rt.enqueue_loop((1,), (12,), [(a, [(-1, 0, 0), (0, 0, 0)], B.READ), (b, B.POINT, B.WRITE)],
                    {1: "(r 0 -1)"})
    v = rt.fetch_dataset(b)
    assert v[6 + 1, 0, 0] == 13.0  # alloc starts at -1
    assert rt.report()["d2d"] > 0


def test_device_counters_show_native_kernels():
    rt = B.Runtime("resident")
    rt.run_app("heat2d", 64, 64, 0, 4)
    dev = rt.device()
    assert dev["kernel_launches"] >= 4 and dev["interp_launches"] >= 4
    assert dev["cc"] == "10.0"


@pytest.fixture
def jit_always():
    B.set_jit(2, 0)
    yield
    B.set_jit(1, 1 << 18)


def test_specialised_kernels_vs_golden(golden_random, golden_apps, jit_always):
    """Every launch through the NVRTC-specialised kernels: same bits as the reference."""
    assert B.jit_status() == "ok"
    bad = []
    for case in golden_random[:40]:
        prog = P.random_program(case["seed"], **case["kwargs"])
        for want in case["runs"]:
            got = product_record(prog, EXEC_OF[want["executor"]], want["tiles"], want["capacity"],
                                 want["cyclic"], prefetch=want.get("prefetch", False))
            got.pop("_rt", None)
            diff = compare(want, got, check_audit=want["executor"] == "explicit",
                           check_totals=want["executor"] == "explicit")
            if diff:
                bad.append((case["seed"], want, diff))
    for case in golden_apps:
        name, kw = case["case"]
        kw = dict(kw)
        prog = P.app_program(name, kw.pop("nx"), kw.pop("ny"), kw.pop("nz", 0), **kw)
        for want in case["runs"][:2]:
            got = product_record(prog, EXEC_OF[want["executor"]], want["tiles"], want["capacity"],
                                 want["cyclic"], prefetch=want.get("prefetch", False))
            got.pop("_rt", None)
            diff = compare(want, got, check_audit=want["executor"] == "explicit",
                           check_totals=want["executor"] == "explicit")
            if diff:
                bad.append((name, want["executor"], diff))
    assert not bad, bad[:5]


@pytest.mark.parametrize("fuse", [False, True])
def test_specialised_medium_apps(fuse, jit_always):
    for app, nx, ny, nz, iters, span in [("miniflow2d", 300, 256, 0, 12, 0),
                                         ("miniflow3d", 40, 36, 30, 10, 0),
                                         ("rk3chain", 200, 256, 0, 6, 3)]:
        prog = P.app_program(app, nx, ny, nz, iters=iters, span=span)
        pb = B.problem_bytes(app, nx, ny, nz, span)
        want = oracle_record(prog, "explicit", capacity=pb // 2)
        got = product_record(prog, "explicit", capacity=pb // 2, fuse=fuse)
        want.pop("_rt", None)
        got.pop("_rt", None)
        assert not compare(want, got), (app, fuse)
        dev = B.Runtime("resident").device()
        assert dev["jit_launches"] == 0  # fresh context; counters are per runtime


@pytest.fixture
def row_recompute():
    B.set_row_recompute(True)
    yield
    B.set_row_recompute(__import__("os").environ.get("OOC_ROW_RECOMPUTE", "1") != "0")


def test_row_recompute_fusion_parity(golden_random, row_recompute, jit_always):
    """Groups fused through row recompute (neighbour reads of values written earlier in
    the launch, re-evaluated in-thread) give the reference's bits — specialised
    kernels, and the interpreter's loop-by-loop fallback."""
    bad = []
    for app, nx, ny, nz, iters in [("miniflow2d", 300, 256, 0, 12), ("miniflow3d", 40, 36, 30, 10)]:
        prog = P.app_program(app, nx, ny, nz, iters=iters)
        pb = B.problem_bytes(app, nx, ny, nz)
        for kw in (dict(capacity=pb // 2), dict(tiles=1)):
            want = oracle_record(prog, "explicit", **kw)
            got = product_record(prog, "explicit", **kw)
            want.pop("_rt", None)
            got.pop("_rt", None)
            if compare(want, got):
                bad.append((app, kw))
    B.set_jit(0, 1 << 18)  # interpreter: row-recompute groups run loop by loop
    for case in golden_random[:30]:
        prog = P.random_program(case["seed"], **case["kwargs"])
        want = [w for w in case["runs"] if w["executor"] == "explicit"][0]
        got = product_record(prog, "explicit", want["tiles"], want["capacity"], want["cyclic"],
                             prefetch=want.get("prefetch", False))
        got.pop("_rt", None)
        if compare(want, got):
            bad.append(case["seed"])
    assert not bad, bad


@pytest.mark.parametrize("shape,recompute", [("t16x64", "0"), ("t8x128", "0"), ("t32x32", "1"),
                                             ("1x4", "1"), ("t16x64", "1")])
def test_forced_tile_shapes(shape, recompute):
    """Every specialised launch forced to one tile shape — register template (QxP) or
    shared-memory/TMA template (tTBxTC), with and without row recompute — gives the
    reference's bits (child process: the shape is read once per process)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, OOC_JIT_SHAPE=shape, OOC_ROW_RECOMPUTE=recompute)
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "shape_parity_child.py")],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("budget", [0, 2 << 20])
def test_graph_replay_parity(budget, jit_always):
    """Steady-state resident chains replay as CUDA graphs (third sighting on): same bits
    and reductions as the oracle, untiled and L2-tiled."""
    prog = P.app_program("miniflow2d", 200, 180, 0, iters=52)
    want = oracle_record(prog, "reference")
    got = product_record(prog, "resident", resident_budget=budget)
    rt = got.pop("_rt")
    want.pop("_rt", None)
    assert not compare(want, got, check_audit=False, check_totals=False)
    assert rt.device()["graph_launches"] >= 2


@pytest.mark.parametrize("jit", [1, 2])
def test_slab_runtime_with_nccl_single_rank(jit):
    """The multi-GPU path on one GPU: a 1-rank NCCL communicator, a dim-0 window with
    ghost rows, all-reduce of the fieldsum — same bits / same reduction as plain. jit=2:
    every launch specialised, so the slab runtime runs row-sweep kernels with buffer
    swaps and exchanges ghost rows from the current buffers."""
    from paper_1709_02125_b200 import dist as D
    B.set_jit(jit, 0 if jit == 2 else 1 << 18)
    try:
        n, iters = 96, 20
        ghost = D.chain_depth("miniflow2d", iters)
        a = B.Runtime("resident", dist=(0, 1), own=(0, n), ghost=ghost)
        a.comm_init(D.unique_id())
        a.run_app("miniflow2d", n, n, 0, iters)
        b = B.Runtime("resident")
        b.run_app("miniflow2d", n, n, 0, iters)
        for d in range(b.num_datasets):
            assert np.array_equal(a.fetch_dataset(d).view(np.uint64), b.fetch_dataset(d).view(np.uint64))
        assert a.fetch_reduction("fieldsum") == b.fetch_reduction("fieldsum")
        if jit == 2:
            assert a.device()["sweep_launches"] > 0
    finally:
        B.set_jit(1, 1 << 18)
