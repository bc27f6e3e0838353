"""Row-sweep planning on CPU (no GPU): which runs of a chain the sweep kernel takes,
their schedules (lags, halos, rings, out-of-place outputs), and that every generated
kernel compiles for sm_100a with NVRTC."""
import pytest

import paper_1709_02125_b200 as B
from oracle import programs as P


@pytest.fixture
def jit_always():
    B.set_jit(2, 0)
    yield
    B.set_jit(1, 1 << 18)


def _chains(prog):
    rt = B.load_program(B.Runtime("plan_only", record=True, tiles=1), prog)
    return rt, range(rt.num_chains())


def test_miniflow2d_timesteps_fuse_into_sweeps(jit_always):
    rt, chains = _chains(P.app_program("miniflow2d", 64, 64, iters=10))
    groups = [g for c in chains for g in rt.chain_sweep_check(c, compile=True)]
    assert groups and all(g["ok"] for g in groups)
    covered = sum(g["loops"] for g in groups)
    assert covered == 141  # 10 iterations x 14 loops + the fieldsum (folded into the last run)
    assert max(g["loops"] for g in groups) >= 14  # at least one whole timestep per launch
    for g in groups:
        pl = g["plan"]
        assert pl["smem"] <= 2 * 56 * 1024 and pl["TC"] + 2 * pl["HC"] == 256
        assert min(pl["lags"]) >= 0 and pl["warm"] >= 0
        for d in pl["datasets"]:
            assert d["oop"] == (d["loaded"] and d["written"])
            assert d["W"] >= pl["K"]
    # temporaries a later run rewrites before reading are not stored (dead stores); the
    # chain's last run stores every dataset it writes
    c1 = rt.chain_sweep_check(max(chains), compile=False)
    assert all(len(g["dead"]) >= 1 for g in c1[:-1]) and c1[-1]["dead"] == []
    assert len(c1[0]["dead"]) == 6
    first = groups[0]["plan"]["datasets"]
    # rho, e, v are read and rewritten: out of place; temporaries are written first
    assert sum(d["oop"] for d in first) == 3


def test_3d_chains_sweep_as_plane_tiles(jit_always):
    """3-D chains become plane-tile sweeps (TMA row copies per tile row) whose kernels
    compile for sm_100a; a whole miniflow3d timestep fits one run."""
    B.set_sweep_3d(False)
    rt, chains = _chains(P.app_program("miniflow3d", 24, 20, 18, iters=3))
    assert all(rt.chain_sweep_check(c, compile=False) == [] for c in chains)  # the switch works
    B.set_sweep_3d(True)
    for app, kw in (("miniflow3d", dict(iters=3)), ("rk3chain3d", dict(iters=3, span=3))):
        rt, chains = _chains(P.app_program(app, 24, 20, 18, **kw))
        runs = [g for c in chains for g in rt.chain_sweep_check(c, compile=True)]
        assert runs and all(g["ok"] for g in runs), runs
        if app == "miniflow3d":
            assert any(g["loops"] >= 14 for g in runs)
            assert all(g["plan"]["tma"] == 1 for g in runs)


def test_random_2d_chains_compile(jit_always):
    n = 0
    for seed in range(60):
        prog = P.random_program(seed, flushes=True, allow_3d=False)
        rt, chains = _chains(prog)
        for c in chains:
            for g in rt.chain_sweep_check(c, compile=True):
                assert g["ok"], (seed, g)
                n += 1
    assert n > 5


def test_sweep_plans_of_other_apps(jit_always):
    """heat2d and the 2-D RK3 chain: whole chains become sweep runs; read-and-rewritten
    datasets are out of place, temporaries in place; lags never negative; every run's
    kernel compiles."""
    for app, kw in (("heat2d", dict(iters=8, span=4)), ("rk3chain", dict(iters=6, span=3))):
        rt, chains = _chains(P.app_program(app, 120, 96, 0, **kw))
        runs = [g for c in chains for g in rt.chain_sweep_check(c, compile=True)]
        assert runs and all(g["ok"] for g in runs), app
        for g in runs:
            pl = g["plan"]
            assert min(pl["lags"]) >= 0 and len(pl["lags"]) == g["loops"]
            assert all(d["oop"] == (d["loaded"] and d["written"]) for d in pl["datasets"])
            assert pl["HC"] >= max(pl["halos"])

