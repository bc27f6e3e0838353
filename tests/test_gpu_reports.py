"""Measured reports in the reference's CSV schemas (proj/src/metrics.cpp:46-79,
proj/src/command.cpp:160-168): the real event timeline of an out-of-core run
accounts for exactly the bytes the audit reports, keeps each queue in order, and
attributes device time to loops (attribute_loop_times, metrics.cpp:14-32) —
without changing a single result bit."""
import csv
import io

import pytest

import paper_1709_02125_b200 as B
from oracle import programs as P
from tests.helpers import compare, oracle_record, product_record

pytestmark = pytest.mark.gpu


def _rows(text):
    lines = [l for l in text.splitlines() if not l.startswith("#")]
    return list(csv.DictReader(io.StringIO("\n".join(lines))))


@pytest.mark.parametrize("app,nx,ny,nz,cyclic,prefetch", [
    ("miniflow2d", 300, 256, 0, True, True),
    ("miniflow2d", 300, 256, 0, False, False),
    ("miniflow3d", 40, 36, 30, True, False),
])
def test_timeline_accounts_for_every_byte(app, nx, ny, nz, cyclic, prefetch):
    prog = P.app_program(app, nx, ny, nz, iters=6)
    want = oracle_record(prog, "explicit", tiles=3, cyclic=cyclic, prefetch=prefetch)
    got = product_record(prog, "explicit", tiles=3, cyclic=cyclic, prefetch=prefetch,
                         timeline=True)
    rt = got.pop("_rt")
    want.pop("_rt", None)
    assert not compare(want, got)

    tl = _rows(rt.timeline_csv())
    assert tl, "no timeline rows"
    rep = _rows(rt.report_csv(app, f"{nx}x{ny}x{nz}", 6))[0]
    by = {k: sum(int(r["bytes"]) for r in tl if r["kind"] == k) for k in ("h2d", "d2h", "d2d", "kernel")}
    assert by["h2d"] == int(rep["uploaded"])
    assert by["d2h"] == int(rep["downloaded"])
    if prefetch:  # consuming the staged tile 0 is a real D2D the audit does not bill
        assert by["d2d"] >= int(rep["d2d"])
    else:
        assert by["d2d"] == int(rep["d2d"])
    assert by["kernel"] == int(rep["total_bytes"])
    # queues are FIFO: in command order each row starts after its predecessor ends
    last = {}
    for r in sorted(tl, key=lambda r: int(r["command_id"])):
        s, e, q = float(r["start"]), float(r["end"]), r["queue"]
        assert s <= e + 1e-9
        assert s >= last.get(q, 0.0) - 2e-6, r
        last[q] = e
    loops = _rows(rt.loops_csv())
    assert len(loops) == len({l["loop"] for l in loops})
    tsum = sum(float(l["time"]) for l in loops)
    kernel_span = max(float(r["end"]) for r in tl if r["kind"] == "kernel")
    assert 0 < tsum <= kernel_span + 1e-6
    assert all(float(l["time"]) >= 0 for l in loops)
    audit = _rows(rt.audit_csv())
    assert sum(int(a["uploaded"]) for a in audit) == int(rep["uploaded"])


def test_timeline_off_records_nothing():
    rt = B.Runtime("resident")
    rt.run_app("heat2d", 64, 64, 0, 4)
    assert rt.timeline_csv() == "command_id,kind,queue,bytes,issue,start,end\n"


def _prefetch_kat():
    """proj/tests/test_device_sim.cpp:316-368: c pure input, a = c, b = a(-1); 3 tiles."""
    p = P.Prog()
    p.declare("c", (0,), (12,), (1,), "(* 0.125 i)")
    p.declare("a", (0,), (12,), (1,), 0.0)
    p.declare("b", (0,), (12,), (1,), 0.0)
    for _ in range(2):
        p.loop((0,), (12,), [("c", P.POINT, P.R), ("a", P.POINT, P.W)], {1: P.r(0)})
        p.loop((0,), (12,), [("a", [(-1, 0, 0), (0, 0, 0)], P.R), ("b", P.POINT, P.W)],
               {1: P.r(0, -1)})
        p.flush()
    p.finish()
    return p.to_dict()


def test_prefetch_kat_second_chain_skips_tile0_upload():
    prog = _prefetch_kat()
    want = oracle_record(prog, "explicit", tiles=3, prefetch=True)
    got = product_record(prog, "explicit", tiles=3, prefetch=True, timeline=True)
    rt = got.pop("_rt")
    want.pop("_rt", None)
    assert not compare(want, got)
    audit = rt.audit()  # rows [dataset, tile, up, down, d2d] of both chains in order
    cut = next(i for i in range(1, len(audit)) if audit[i][0] < audit[i - 1][0])
    second = audit[cut:]
    assert sum(r[2] for r in audit[:cut] if r[1] == 0) == 72
    assert sum(r[2] for r in second if r[1] == 0) == 0
    plain = product_record(prog, "explicit", tiles=3)
    plain.pop("_rt")
    assert plain["buffers"] == got["buffers"]
