"""BASELINE configs 2-5 on one B200: in-core (untiled and L2-tiled) vs out-of-core at
1.5x and 3x the device budget, 2-D and 3-D workloads. One JSON line per run.

    python scripts/suite.py [config ...]     (default: all)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1709_02125_b200 as B  # noqa: E402

# app, nx, ny, nz, iterations per step (= one chain), span
WORK = {
    "miniflow2d": ("miniflow2d", 15360, 15360, 0, 10, 0),
    "miniflow3d": ("miniflow3d", 600, 600, 600, 10, 0),
    "rk3chain3d": ("rk3chain3d", 700, 700, 700, 3, 3),
    # high-reuse chains: ten RK3 timesteps per chain
    "rk3chain3d_s10": ("rk3chain3d", 640, 640, 640, 10, 10),
    "rk3chain_s10": ("rk3chain", 15360, 15360, 0, 10, 10),
}


def run(app_key, executor, steps=3, warmup=5, **kw):
    app, nx, ny, nz, per, span = WORK[app_key]
    rt = B.Runtime(executor, **kw)
    t0 = time.perf_counter()
    rt.declare_app(app, nx, ny, nz, span)
    t_decl = time.perf_counter() - t0
    rt.app_iterations(app, nx, ny, nz, 0, per * warmup, span, cyclic=CYCLIC[0])
    rt.sync()
    r0 = rt.report()
    m0 = rt.mark()
    t0 = time.perf_counter()
    rt.app_iterations(app, nx, ny, nz, per * warmup, per * (warmup + steps), span, cyclic=CYCLIC[0])
    m1 = rt.mark()
    rt.sync()
    wall = time.perf_counter() - t0
    dev_s = rt.elapsed(m0, m1)
    r1 = rt.report()
    nbytes = r1["total_bytes"] - r0["total_bytes"]
    out = {"app": app_key, "executor": executor, "steps": steps,
           "problem_bytes": B.problem_bytes(app, nx, ny, nz, span),
           "metric_bytes": nbytes, "device_s": dev_s, "wall_s": wall,
           "GBps_device": nbytes / dev_s / 1e9, "GBps_wall": nbytes / wall / 1e9,
           "tiles": r1["tiles"], "uploaded": r1["uploaded"] - r0["uploaded"],
           "downloaded": r1["downloaded"] - r0["downloaded"], "d2d": r1["d2d"] - r0["d2d"],
           "declare_s": t_decl, "launches": rt.device()["kernel_launches"],
           # per-chain reuse of the link bytes: metric bytes per byte moved over PCIe
           "reuse": nbytes / max(1, (r1["uploaded"] - r0["uploaded"]) + (r1["downloaded"] - r0["downloaded"]))}
    rt.close()
    return out


CYCLIC = [False]


def main():
    which = sys.argv[1:] or ["2", "3", "4", "5"]
    lines = []
    if "2" in which:  # in-core, tiled vs untiled
        # tiled on chip: row sweeps (CTA segments are skewed tiles of whole timesteps)
        lines.append(dict(config=2, mode="in-core tiled: row sweeps through shared memory",
                          **run("miniflow2d", "resident")))
        B.set_sweep(False)  # untiled: every loop group sweeps the whole mesh through HBM
        lines.append(dict(config=2, mode="in-core untiled: fused loop-group launches",
                          **run("miniflow2d", "resident")))
        lines.append(dict(config=2, mode="in-core tiled through L2: reference skew tiles (slot <= 96 MB)",
                          **run("miniflow2d", "resident", resident_budget=96 << 20, steps=1, warmup=1)))
        B.set_sweep(True)
    for cfg, app, cyc in (("3", "miniflow2d", False), ("3", "miniflow2d", True),
                          ("4", "miniflow3d", True), ("5", "rk3chain3d", False),
                          ("5s10", "rk3chain3d_s10", False), ("5s10", "rk3chain3d_s10", True),
                          ("2s10", "rk3chain_s10", False), ("2s10", "rk3chain_s10", True)):
        if cfg not in which:
            continue
        CYCLIC[0] = cyc
        pb = B.problem_bytes(*[WORK[app][i] for i in (0, 1, 2, 3)], WORK[app][5])
        base = run(app, "resident")
        lines.append(dict(config=cfg, mode="in-core baseline", cyclic=cyc, **base))
        # span-10 3-D chains: the planner's smallest 3-slot size exceeds a third of the
        # problem (InfeasibleError, recorded), so they also run at half
        for ratio in ((1.5, 3.0) if cfg == "3" else (3.0, 2.0) if cfg == "5s10" else (3.0,)):
            try:
                r = run(app, "explicit", capacity=int(pb / ratio))
                r.update(config=cfg, mode=f"out-of-core {ratio}x (capacity = problem/{ratio})",
                         cyclic=cyc, ooc_over_incore=r["GBps_wall"] / base["GBps_device"])
            except Exception as e:  # noqa: BLE001
                r = {"config": cfg, "app": app, "ratio": ratio, "error": str(e)}
            lines.append(r)
        CYCLIC[0] = False
    for l in lines:
        print(json.dumps(l), flush=True)


if __name__ == "__main__":
    main()
