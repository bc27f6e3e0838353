"""GPU parity of the row-sweep kernels (csrc/device/sweep.cu): runs of 2-D loops —
whole miniflow2d timesteps and random stencil chains — streamed through shared-memory
rings in one launch, outputs written out of place and the buffers swapped. Fields
must be bit-identical to the oracle / the reference's golden fixtures, reductions
within 1e-12 (north_star)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1709_02125_b200 as B
from oracle import programs as P
from tests.helpers import compare, oracle_record, product_record

pytestmark = pytest.mark.gpu


@pytest.fixture
def jit_always():
    B.set_jit(2, 0)
    yield
    B.set_jit(1, 1 << 18)


def _resident_vs_oracle(prog, **kw):
    want = oracle_record(prog, "reference")
    got = product_record(prog, "resident", **kw)
    rt = got.pop("_rt")
    want.pop("_rt", None)
    return compare(want, got, check_audit=False, check_totals=False), rt


@pytest.mark.parametrize("app,nx,ny,iters,span", [
    ("miniflow2d", 300, 256, 12, 0),
    ("miniflow2d", 517, 263, 23, 0),
    ("miniflow2d", 64, 700, 10, 0),
    ("heat2d", 300, 256, 12, 4),
    ("heat2d", 257, 129, 9, 0),
    ("rk3chain", 200, 256, 6, 3),
])
def test_sweep_apps_vs_oracle(app, nx, ny, iters, span, jit_always):
    prog = P.app_program(app, nx, ny, 0, iters=iters, span=span)
    diff, rt = _resident_vs_oracle(prog)
    assert not diff, diff
    assert rt.device()["sweep_launches"] > 0


@pytest.mark.parametrize("app,nx,ny,nz,iters,span", [
    ("miniflow3d", 40, 36, 30, 12, 0),
    ("miniflow3d", 70, 45, 66, 10, 0),
    ("rk3chain3d", 32, 30, 28, 3, 3),
    ("rk3chain3d", 60, 41, 37, 2, 1),
])
def test_sweep_3d_apps_vs_oracle(app, nx, ny, nz, iters, span, jit_always):
    """3-D chains as plane-tile sweeps (threads over a dim-1 x column tile, rings of plane
    tiles, dim-1 and column halos recomputed): bit-identical to the oracle."""
    B.set_sweep_3d(True)
    try:
        prog = P.app_program(app, nx, ny, nz, iters=iters, span=span)
        diff, rt = _resident_vs_oracle(prog)
        assert not diff, diff
        assert rt.device()["sweep_launches"] > 0
    finally:
        B.set_sweep_3d(True)


def test_sweep_random_3d_chains_vs_oracle(jit_always):
    """Random 3-D chains (mixed stencils along all three dimensions, read-write loops,
    reductions) on meshes larger than a plane tile: several tiles per plane, interior
    (fast, unrolled) and edge (predicated) tiles, against the oracle bit for bit."""
    swept = 0
    for seed in range(24):
        prog = P.random_program(1000 + seed, force_ndim=3, min_size=20, max_size=44, max_3d=44, flushes=True)
        diff, rt = _resident_vs_oracle(prog)
        assert not diff, (seed, diff)
        swept += rt.device()["sweep_launches"]
    assert swept > 0


def test_sweep_random_programs_vs_golden(golden_random, jit_always):
    """Random 2-D chains (mixed stencils, ranges, read-write loops, flushes, reductions)
    through the resident executor: the reference's golden buffers and reductions."""
    bad, swept = [], 0
    for case in golden_random:
        prog = P.random_program(case["seed"], **case["kwargs"])
        for want in case["runs"]:
            if want["executor"] != "reference":
                continue
            got = product_record(prog, "resident")
            rt = got.pop("_rt", None)
            if rt is not None:
                swept += rt.device()["sweep_launches"]
            diff = compare(want, got, check_audit=False, check_totals=False)
            if diff:
                bad.append((case["seed"], diff))
    assert not bad, bad[:5]
    assert swept > 0


def test_sweep_large_random_programs(jit_always):
    """Random 2-D chains on 300-700 point meshes (partial ranges, read-write loops, mixed
    stencils, flushes, reductions): enough rows and columns for interior strips, so the
    predicate-free fast steps, register forwarding and carries run against the oracle."""
    bad, swept = [], 0
    for seed in range(40):
        prog = P.random_program(seed, max_loops=12, min_size=300, max_size=700, allow_3d=False, flushes=True)
        want = oracle_record(prog, "reference")
        got = product_record(prog, "resident")
        rt = got.pop("_rt", None)
        want.pop("_rt", None)
        if rt is not None:
            swept += rt.device()["sweep_launches"]
        diff = compare(want, got, check_audit=False, check_totals=False)
        if diff:
            bad.append((seed, diff))
    assert not bad, bad[:5]
    assert swept > 0


def test_sweep_graph_replay_flips(jit_always):
    """Captured chains replay with the recorded buffer swaps: 112 iterations (an odd number
    of swaps per chain, so consecutive chains alternate between two graphs) stay
    bit-exact."""
    prog = P.app_program("miniflow2d", 200, 180, 0, iters=112)
    diff, rt = _resident_vs_oracle(prog)
    assert not diff, diff
    dev = rt.device()
    assert dev["graph_launches"] >= 2 and dev["sweep_launches"] > 0


def test_sweep_fetch_between_chains(jit_always):
    """fetch_dataset in the middle of a run reads the current buffer of a swapped pair."""
    from oracle import ooc_oracle as O
    n = 160
    rt = B.Runtime("resident")
    rt.run_app("miniflow2d", n, n, 0, 20)
    ref = O.Runtime("reference")
    prog = P.app_program("miniflow2d", n, n, 0, iters=20)
    O.load_program(ref, prog)
    for d in range(rt.num_datasets):
        got = rt.fetch_dataset(d)
        assert np.array_equal(np.asarray(got).view(np.uint64), ref.mesh[d].host.view(np.uint64)), d
    assert rt.device()["sweep_launches"] > 0


@pytest.mark.parametrize("K,P_,smem,rc", [("1", "1", "60000", "128"), ("4", "2", "200000", "256"),
                                          ("2", "3", "40000", "64"), ("8", "1", "220000", "128"),
                                          ("1", "2", "30000", "64")])
def test_sweep_variants(K, P_, smem, rc):
    """Rows per step K, prefetch depth P, ring width and the shared-memory budget (which
    sets how many loops one sweep spans) change the schedule, never the bits (child
    process: read once per process)."""
    env = dict(os.environ, OOC_SWEEP_K=K, OOC_SWEEP_P=P_, OOC_SWEEP_SMEM=smem, OOC_SWEEP_RC=rc)
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "sweep_parity_child.py")],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("env", [
    {"OOC_SWEEP_EDGEFIRST": "0", "OOC_SWEEP_MASKED": "0"},
    {"OOC_SWEEP_RC": "64", "OOC_SWEEP_SMEM": "60000", "OOC_SWEEP_NSEG": "3"},
    {"OOC_SWEEP_RC": "64", "OOC_SWEEP_SMEM": "60000", "OOC_SWEEP_MASKED": "0"},
])
def test_sweep_schedule_variants(env):
    """CTA scheduling — column-edge strips dispatched first, masked fast steps on edge
    strips, forced segment counts — with narrow rings (many strips, so most CTAs are
    edge-first reordered and several take masked steps) never changes the bits."""
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "sweep_parity_child.py")],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def test_sweep_build_failure_falls_back():
    """A row-sweep kernel that cannot be built (forced by OOC_SWEEP_FAIL_BUILD) falls back
    to the fused loop-group launches: bits unchanged, each loop's bytes billed once."""
    env = dict(os.environ, OOC_SWEEP_FAIL_BUILD="1")
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "sweep_fallback_child.py")],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "row sweep unavailable" in r.stderr
