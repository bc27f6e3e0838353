"""Slab decomposition on CPU (world_size 2 and 3, gloo): the product's decomposition
(window clipping of datasets and loops, ghost depth, ghost-band exchange plan,
owned-row reductions — csrc/host/runtime.cpp) is executed with the numpy oracle on
each rank's local mesh, ghost bands exchanged over gloo exactly as the plan says,
reductions all-reduced; owned rows must equal the single-domain oracle bit for bit
and reductions within 1e-12. The GPU path runs the same plan over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1709_02125_b200 as B
from oracle import ooc_oracle as O
from oracle import programs as P
from paper_1709_02125_b200 import dist as D

CASES = {
    "miniflow2d": dict(nx=60, ny=40, nz=0, iters=12, span=0),
    "rk3chain": dict(nx=54, ny=30, nz=0, iters=6, span=3),
    "miniflow3d": dict(nx=24, ny=12, nz=10, iters=10, span=0),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _global_rows(app, kw):
    """Dim-0 core rows of the app's datasets (owned rows are split over these)."""
    if app.startswith("rk3"):
        pad = 3 * (kw["span"] or 1) - 1
        return -pad, kw["nx"] + pad
    return 0, kw["nx"]


def _worker(rank, world, port, app, out_q):
    os.environ["OMP_NUM_THREADS"] = "1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        kw = CASES[app]
        nd = 3 if app.endswith("3d") else 2
        ghost = D.chain_depth(app, kw["iters"], kw["span"], nd)
        r0, r1 = _global_rows(app, kw)
        own = D.slab(rank, world, r1 - r0, r0)
        rt = B.Runtime("plan_only", record=True, tiles=1, dist=(rank, world), own=own, ghost=ghost)
        rt.run_app(app, kw["nx"], kw["ny"], kw["nz"], kw["iters"], kw["span"])
        prog = P.app_program(app, kw["nx"], kw["ny"], kw["nz"], iters=kw["iters"], span=kw["span"])
        spec = {d["name"]: d for d in prog["datasets"]}
        ort = O.Runtime("reference")
        ids = {}
        names = [None] * rt.num_datasets
        for jd in prog["datasets"]:
            names[rt.find(jd["name"])] = jd["name"]
        for d, name in enumerate(names):
            info = rt.dataset_info(d)
            h = spec[name]["halo"]
            halo = [h] * nd if isinstance(h, int) else list(h)
            lo = [info["lo"][k] + halo[k] for k in range(nd)]
            hi = [info["hi"][k] - halo[k] for k in range(nd)]
            ids[name] = ort.declare(name, O.Ext.make(nd, lo, hi), halo, 8, spec[name]["fill"])
        reductions = {}
        for c in range(rt.num_chains()):
            for jl in rt.chain_export(c):
                args = [O.Arg(ids[a["dataset"]], [tuple(o) for o in a["offsets"]], a["mode"])
                        for a in jl["args"]]
                loop = O.Loop(O.Ext.make(nd, jl["lo"], jl["hi"]), args,
                              [(int(k), O.parse_prefix(v)) for k, v in sorted(jl["writes"].items())])
                if "reduction" in jl:
                    r = jl["reduction"]
                    loop.reduce_op, loop.reduce_tree, loop.reduce_name = (
                        r["op"], O.parse_prefix(r["expr"]), r["name"])
                O.validate_loop(ort.mesh, loop)
                acc = O.reduce_identity(loop.reduce_op) if loop.reduce_op else None
                acc = O.apply_loop(ort.mesh, loop, loop.range, acc)
                if loop.reduce_op:
                    import torch
                    t = torch.tensor([acc], dtype=torch.float64)
                    dist.all_reduce(t, op=dist.ReduceOp.SUM)
                    reductions[loop.reduce_name] = float(t.item())
            # ghost-band exchange, exactly as the product's plan prescribes
            import torch
            reqs, recvs = [], []
            for hx in rt.dist_plan(c)["halos"]:
                ds = ort.mesh[ids[hx["dataset"]]]
                a0 = ds.alloc().lo[0]
                for side, peer in (("left", rank - 1), ("right", rank + 1)):
                    s0, s1 = hx["send_" + side]
                    q0, q1 = hx["recv_" + side]
                    if peer < 0 or peer >= world:
                        continue
                    if s1 > s0:
                        reqs.append(dist.isend(torch.from_numpy(
                            np.ascontiguousarray(ds.host[s0 - a0:s1 - a0])), peer))
                    if q1 > q0:
                        buf = torch.empty(ds.host[q0 - a0:q1 - a0].shape, dtype=torch.float64)
                        reqs.append(dist.irecv(buf, peer))
                        recvs.append((ds, q0 - a0, q1 - a0, buf))
            for r in reqs:
                r.wait()
            for ds, a, b, buf in recvs:
                ds.host[a:b] = buf.numpy()
        # owned rows (plus the global edge rows at the first/last rank)
        result = {}
        for name, d in ids.items():
            ds = ort.mesh[d]
            a = ds.alloc()
            lo = own[0] if rank > 0 else a.lo[0]
            hi = own[1] if rank + 1 < world else a.hi[0]
            result[name] = (lo, ds.host[lo - a.lo[0]:hi - a.lo[0]].copy())
        out_q.put((rank, result, reductions, ghost))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("app", sorted(CASES))
def test_slab_decomposition_matches_single_domain(app, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, app, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    kw = CASES[app]
    prog = P.app_program(app, kw["nx"], kw["ny"], kw["nz"], iters=kw["iters"], span=kw["span"])
    ref = O.load_program(O.Runtime("reference"), prog)
    for rank, result, reductions, ghost in parts:
        assert ghost > 0
        for name, (lo, rows) in result.items():
            ds = ref.mesh[ref.find(name)]
            a0 = ds.alloc().lo[0]
            want = ds.host[lo - a0:lo - a0 + rows.shape[0]]
            assert np.array_equal(rows.view(np.uint64), want.view(np.uint64)), (app, rank, name)
        for name, v in reductions.items():
            assert abs(v - ref.reductions[name]) <= 1e-12 * abs(ref.reductions[name])
