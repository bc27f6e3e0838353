"""Parity at scale against the unmodified reference (oracle/_ref/libooc_ref.so, built from
/root/reference and shipped with the repo): miniflow2d at 2048 x 2048 — in core (whole
timesteps as row-sweep kernels, multi-strip multi-segment grids, CUDA-graph replays) and
out of core (capacity = problem/3, cyclic, prefetch) — fields bit for bit, the fieldsum
within 1e-12 of the reference's sequential fold. bench.py repeats the check at the
benched 15360 x 15360 (its "parity" block)."""
import os

import numpy as np
import pytest

import paper_1709_02125_b200 as B
from oracle import refo

N = 2048
ITERS = 30  # three 10-iteration chains with a fieldsum each


@pytest.fixture(scope="module")
def reference():
    if not refo.available():
        pytest.skip("oracle/_ref/libooc_ref.so not built")
    ref = refo.RefRuntime("reference", openmp=True)
    ref.run_app("miniflow2d", N, N, ITERS)
    yield ref
    ref.close()


def _check(rt, ref, allow_stale=False, exact=False):
    names = ref.datasets()
    checked = 0
    for d in range(rt.num_datasets):
        if allow_stale and rt.dataset_info(d)["stale"]:
            continue
        got = np.ascontiguousarray(rt.host(d)).reshape(-1)
        want = ref.host_view(d)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), names[d]
        checked += 1
    a, b = rt.fetch_reduction("fieldsum"), ref.fetch_reduction("fieldsum")
    if exact:
        assert a.hex() == b.hex(), (a, b)
    assert abs(a - b) <= 1e-12 * abs(b), (a, b)
    return checked


@pytest.mark.gpu
def test_incore_sweeps_2048_vs_reference(reference):
    rt = B.Runtime("resident")
    rt.run_app("miniflow2d", N, N, 0, ITERS)
    rt.finish()
    assert _check(rt, reference) == 10
    assert rt.device()["sweep_launches"] > 0
    rt.close()


@pytest.mark.gpu
def test_out_of_core_2048_vs_reference(reference):
    cap = B.problem_bytes("miniflow2d", N, N) // 3
    rt = B.Runtime("explicit", capacity=cap, prefetch=True)
    rt.run_app("miniflow2d", N, N, 0, ITERS, cyclic=True)
    rt.finish()
    assert _check(rt, reference, allow_stale=True) >= 4  # rho, e, v, gamma stay fresh
    rt.close()


@pytest.mark.gpu
def test_exact_reductions_2048_vs_reference(reference):
    """Exact mode: the fieldsum folded in the reference's row-major order, bit for bit,
    while the non-reducing loops still run as row sweeps."""
    rt = B.Runtime("resident", exact_reductions=True)
    rt.run_app("miniflow2d", N, N, 0, ITERS)
    rt.finish()
    assert _check(rt, reference, exact=True) == 10
    assert rt.device()["sweep_launches"] > 0
    rt.close()
    cap = B.problem_bytes("miniflow2d", N, N) // 3
    rt = B.Runtime("explicit", capacity=cap, prefetch=True, exact_reductions=True)
    rt.run_app("miniflow2d", N, N, 0, ITERS, cyclic=True)
    rt.finish()
    assert _check(rt, reference, allow_stale=True, exact=True) >= 4
    rt.close()


@pytest.mark.gpu
def test_exact_reductions_refuse_slabs():
    rt = B.Runtime("resident", dist=(0, 2), own=(0, 64), ghost=4, exact_reductions=True)
    with pytest.raises(B.ValidationError, match="exact"):
        rt.run_app("miniflow2d", 128, 128, 0, 2)
        rt.finish()
    rt.close()
