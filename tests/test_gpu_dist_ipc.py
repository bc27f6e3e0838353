"""Slab decomposition with real neighbour exchanges on ONE GPU: 2 and 3 processes, each a
rank running the product's kernels on its dim-0 slab, ghost bands pulled out of the
neighbours' CUDA-IPC-mapped outboxes after every chain (the transport NCCL cannot provide
when ranks share a GPU), reductions combined across ranks. No kernel ever waits on
another rank (the ranks meet in a host barrier only). Owned rows must equal the
single-domain run bit for bit and the fieldsum match within 1e-12 — resident (row-sweep
kernels) and out of core (each rank streams its own slab through 3 slots under its own
capacity cap, ghost rows refreshed host to host)."""
import os
import subprocess
import sys
import uuid

import numpy as np
import pytest

import paper_1709_02125_b200 as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = os.path.join(ROOT, "tests", "dist_ipc_child.py")

CASES = {  # app: (nx, ny, nz, iters, span)
    "miniflow2d": (240, 160, 0, 30, 0),
    "rk3chain": (200, 120, 0, 9, 3),
    "miniflow3d": (40, 24, 20, 20, 0),
}


def _run_ranks(world, executor, app, tmp_path, cyclic=False):
    nx, ny, nz, iters, span = CASES[app]
    name = uuid.uuid4().hex[:16]
    env = dict(os.environ, OOC_IPC_TIMEOUT="120", OOC_TEST_CYCLIC="1" if cyclic else "0")
    procs, outs = [], []
    for r in range(world):
        out = str(tmp_path / f"rank{r}.npz")
        outs.append(out)
        procs.append(subprocess.Popen([sys.executable, CHILD, str(r), str(world), name, executor, app, str(nx), str(ny),
                                       str(nz), str(iters), str(span), out],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    logs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(o)
        assert p.returncode == 0, o[-3000:]
    return [dict(np.load(o)) for o in outs]


def _single_domain(executor, app, cyclic=False):
    nx, ny, nz, iters, span = CASES[app]
    B.set_jit(2, 0)
    try:
        rt = B.Runtime("resident")
        rt.run_app(app, nx, ny, nz, iters, span)
        full = []
        for d in range(rt.num_datasets):
            info = rt.dataset_info(d)
            full.append((info["lo"][0], rt.fetch_dataset(d)))
        try:
            red = rt.fetch_reduction("fieldsum")
        except B.OocError:
            red = None
        rt.close()
    finally:
        B.set_jit(1, 1 << 18)
    return full, red


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("executor", ["resident", "explicit"])
@pytest.mark.parametrize("app", sorted(CASES))
def test_slab_ranks_on_one_gpu_match_single_domain(app, executor, world, tmp_path):
    parts = _run_ranks(world, executor, app, tmp_path)
    full, red = _single_domain(executor, app)
    for rank, part in enumerate(parts):
        assert part["ghost"][0] > 0
        if world > 1:
            assert part["comm_bytes"][0] > 0, "no ghost band moved"
        for d, (a0, want) in enumerate(full):
            lo, hi = part[f"rows{d}"]
            got = part[f"data{d}"]
            assert got.shape[0] == hi - lo
            assert np.array_equal(got.view(np.uint64), want[lo - a0:hi - a0].view(np.uint64)), (app, executor, rank, d)
        if "fieldsum" in part and red is not None:
            assert abs(part["fieldsum"][0] - red) <= 1e-12 * abs(red), (part["fieldsum"][0], red)
    if executor == "resident" and app != "miniflow3d":
        assert all(p["sweeps"][0] > 0 for p in parts), "row-sweep kernels did not run on the slabs"


@pytest.mark.gpu
@pytest.mark.parametrize("executor", ["resident", "explicit"])
def test_four_ranks_interior_slabs(executor, tmp_path):
    """Four ranks: two interior slabs exchange with both neighbours every chain."""
    parts = _run_ranks(4, executor, "miniflow2d", tmp_path)
    full, red = _single_domain(executor, "miniflow2d")
    for rank, part in enumerate(parts):
        assert part["comm_bytes"][0] > 0
        for d, (a0, want) in enumerate(full):
            lo, hi = part[f"rows{d}"]
            assert np.array_equal(part[f"data{d}"].view(np.uint64), want[lo - a0:hi - a0].view(np.uint64)), (rank, d)
        assert abs(part["fieldsum"][0] - red) <= 1e-12 * abs(red)


@pytest.mark.gpu
def test_slab_out_of_core_cyclic_ranks(tmp_path):
    """Out-of-core slabs with cyclic temporaries: the fields the ranks keep on the host
    (non-stale) equal the single-domain run; stale temporaries are never exchanged."""
    parts = _run_ranks(2, "explicit", "miniflow2d", tmp_path, cyclic=True)
    full, red = _single_domain("explicit", "miniflow2d")
    stale_seen = False
    for part in parts:
        for d, (a0, want) in enumerate(full):
            if part[f"stale{d}"][0]:
                stale_seen = True
                continue
            lo, hi = part[f"rows{d}"]
            assert np.array_equal(part[f"data{d}"].view(np.uint64), want[lo - a0:hi - a0].view(np.uint64)), d
        assert abs(part["fieldsum"][0] - red) <= 1e-12 * abs(red)
    assert stale_seen
