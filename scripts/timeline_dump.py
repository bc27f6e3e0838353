"""Measured command timeline of an out-of-core run (reference CSV schemas) plus a
queue-occupancy summary: how much of the makespan each stream is busy and how much
of the H2D / D2H traffic hides under kernels.

    python scripts/timeline_dump.py [app nx ny nz iters ratio] -> gpurun_out/timeline_*.csv
"""
import json
import time
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1709_02125_b200 as B  # noqa: E402


def busy(iv):
    iv = sorted(iv)
    tot, cur = 0.0, None
    for s, e in iv:
        if cur is None or s > cur[1]:
            if cur:
                tot += cur[1] - cur[0]
            cur = [s, e]
        else:
            cur[1] = max(cur[1], e)
    if cur:
        tot += cur[1] - cur[0]
    return tot


def main():
    a = sys.argv[1:]
    app = a[0] if a else "miniflow2d"
    nx, ny, nz = (int(x) for x in (a[1:4] if len(a) >= 4 else (7680, 7680, 0)))
    iters = int(a[4]) if len(a) > 4 else 30
    ratio = float(a[5]) if len(a) > 5 else 3.0
    pb = B.problem_bytes(app, nx, ny, nz)
    per = 10  # iterations per chain (one bench step)

    def session(timeline):
        rt = B.Runtime("explicit", capacity=int(pb / ratio), prefetch=True, timeline=timeline)
        rt.declare_app(app, nx, ny, nz)
        rt.app_iterations(app, nx, ny, nz, 0, per * 5)  # warm-up: JIT compile + tune
        rt.set_cyclic_flag(True)
        rt.sync()
        n0 = len(rt.timeline_csv().splitlines()) - 1
        t0 = time.perf_counter()
        rt.app_iterations(app, nx, ny, nz, per * 5, per * 5 + iters, cyclic=True)
        rt.sync()
        return rt, n0, time.perf_counter() - t0

    plain, _, wall_plain = session(False)
    plain.close()
    rt, n0, wall = session(True)
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    tag = f"{app}_{nx}x{ny}x{nz}_r{ratio:g}"
    tl = rt.timeline_csv()
    for name, text in (("timeline", tl), ("report", rt.report_csv(app, f"{nx}x{ny}x{nz}", iters)),
                       ("loops", rt.loops_csv()), ("audit", rt.audit_csv())):
        with open(os.path.join(out, f"{name}_{tag}.csv"), "w") as f:
            f.write(text)
    rows = [r.split(",") for r in tl.splitlines()[1 + n0:]]
    span = max(float(r[6]) for r in rows) - min(float(r[5]) for r in rows)
    summ = {"app": app, "size": [nx, ny, nz], "iters": iters, "ratio": ratio, "makespan_s": span,
            "commands": len(rows), "wall_s": wall, "wall_s_without_timeline": wall_plain,
            "metric_GBps_wall": sum(int(r[3]) for r in rows if r[1] == "kernel") / wall / 1e9}
    for kind in ("h2d", "d2h", "d2d", "kernel"):
        iv = [(float(r[5]), float(r[6])) for r in rows if r[1] == kind]
        b = sum(int(r[3]) for r in rows if r[1] == kind)
        summ[kind] = {"n": len(iv), "bytes": b, "busy_s": busy(iv), "busy_frac": busy(iv) / span,
                      "GBps_while_busy": b / busy(iv) / 1e9 if iv and busy(iv) > 0 else None}
    print(json.dumps(summ))
    with open(os.path.join(out, f"timeline_{tag}.json"), "w") as f:
        json.dump(summ, f, indent=1)


if __name__ == "__main__":
    main()
