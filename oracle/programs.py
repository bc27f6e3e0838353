"""ORACLE — TEST INFRASTRUCTURE ONLY.

Program builders in the reference's chain-file JSON format
(proj/src/chain_file.cpp:58-162, extended with an "ops" list; see
oracle/ref/ref_capi.cpp). One program text drives all three implementations:
the unmodified reference (oracle/refo.py), the numpy restatement
(oracle/ooc_oracle.py) and the product (paper_1709_02125_b200.load_program).

* heat2d / miniflow2d / rk3chain restate proj/src/apps.cpp:36-213 loop for loop
  (fills are written as coordinate expressions that evaluate in the same order
  as the C++ lambdas, so buffers are bit-identical to run_app's).
* miniflow3d / rk3chain3d are the 3-D analogues needed by BASELINE configs 4-5
  (CloverLeaf 3D, OpenSBLI TGV 3D). The reference bundles only 2-D apps
  (proj/include/ooc/apps.hpp:10); these are authored against its own API, so
  the reference still runs them as the oracle. The product's C++ apps
  (csrc/host/apps.cpp) define the identical chains.
* random_program mirrors the distribution of the reference's randomised test
  fixture (proj/tests/support.hpp:17-138) with a portable Python RNG.
"""
from __future__ import annotations

import json
import random
from typing import Dict, List, Sequence

# ----------------------------------------------------------------- expressions


def _num(v: float) -> str:
    s = repr(float(v))
    return s


def c(v):
    return _num(v)


def r(arg, o0=0, o1=0, o2=0):
    return f"(r {arg} {o0} {o1} {o2})"


def add(a, b):
    return f"(+ {a} {b})"


def sub(a, b):
    return f"(- {a} {b})"


def mul(a, b):
    return f"(* {a} {b})"


def div(a, b):
    return f"(/ {a} {b})"


def mn(a, b):
    return f"(min {a} {b})"


def mx(a, b):
    return f"(max {a} {b})"


POINT = [(0, 0, 0)]


def star(ndim, radius=1):  # stencil.hpp:28-41
    offs = [(0, 0, 0)]
    for d in range(ndim):
        for o in range(-radius, radius + 1):
            if o == 0:
                continue
            p = [0, 0, 0]
            p[d] = o
            offs.append(tuple(p))
    return offs


def line(dim, radius=1):  # stencil.hpp:20-27
    offs = []
    for o in range(-radius, radius + 1):
        p = [0, 0, 0]
        p[dim] = o
        offs.append(tuple(p))
    return offs


class Prog:
    def __init__(self):
        self.datasets: List[dict] = []
        self.stencils: Dict[tuple, str] = {}
        self.ops: List[dict] = []
        self.ndim = None

    def declare(self, name, lo, hi, halo, fill=0.0, elem_bytes=8):
        self.ndim = len(lo)
        self.datasets.append({"name": name, "core": {"lo": list(lo), "hi": list(hi)},
                              "halo": list(halo)[:len(lo)], "elem_bytes": elem_bytes,
                              "fill": fill})
        return name

    def _stencil(self, offsets):
        key = tuple(tuple(o) for o in offsets)
        if key == ((0, 0, 0),):
            return "point"
        if key not in self.stencils:
            self.stencils[key] = f"s{len(self.stencils)}"
        return self.stencils[key]

    def loop(self, lo, hi, args, writes=None, reduction=None):
        """args: [(dataset, offsets, mode)], writes: {arg: expr}, reduction: (op, expr, name)."""
        jl = {"op": "loop", "range": {"lo": list(lo), "hi": list(hi)},
              "args": [{"dataset": d, "stencil": self._stencil(o), "mode": m} for d, o, m in args],
              "kernel": {}}
        if writes:
            jl["kernel"]["writes"] = {str(k): v for k, v in writes.items()}
        if reduction:
            jl["kernel"]["reduction"] = {"op": reduction[0], "expr": reduction[1],
                                         "name": reduction[2]}
        self.ops.append(jl)

    def flush(self):
        self.ops.append({"op": "flush"})

    def cyclic(self, on=True):
        self.ops.append({"op": "cyclic", "on": bool(on)})

    def finish(self):
        self.ops.append({"op": "finish"})

    def to_dict(self):
        nd = self.ndim or 3
        return {"datasets": self.datasets,
                "stencils": [{"name": n, "offsets": [list(o)[:nd] for o in k]}
                             for k, n in self.stencils.items()],
                "ops": self.ops}

    def to_json(self):
        return json.dumps(self.to_dict())


R, W, RW = "READ", "WRITE", "READ_WRITE"

# ----------------------------------------------------------------- 2-D apps (apps.cpp)


def avg4(arg):  # apps.cpp:25-28
    return mul(c(0.25), add(add(r(arg, -1, 0), r(arg, 1, 0)), add(r(arg, 0, -1), r(arg, 0, 1))))


def star5(arg):  # apps.cpp:30-34
    return mul(c(0.2), add(add(add(r(arg, -1, 0), r(arg, 1, 0)), add(r(arg, 0, -1), r(arg, 0, 1))),
                           r(arg, 0, 0)))


def heat2d(nx, ny, iters, span=0, cyclic=False):  # apps.cpp:36-55
    p = Prog()
    p.declare("u", (0, 0), (nx, ny), (1, 1), "(+ (+ 1.0 (* 0.001 i)) (* 0.002 j))")
    p.declare("tmp", (0, 0), (nx, ny), (1, 1), 0.0)
    if cyclic:
        p.cyclic(True)
    s5 = star(2)
    for it in range(iters):
        src, dst = ("u", "tmp") if it % 2 == 0 else ("tmp", "u")
        p.loop((1, 1), (nx - 1, ny - 1), [(src, s5, R), (dst, POINT, W)], {1: avg4(0)})
        if span > 0 and (it + 1) % span == 0:
            p.flush()
    p.finish()
    return p.to_dict()


def miniflow2d(nx, ny, iters, span=0, cyclic=False):  # apps.cpp:57-154
    p = Prog()
    core_lo, core_hi = (0, 0), (nx, ny)
    wlo, whi = (-1, -1), (nx + 1, ny + 1)
    p.declare("rho", core_lo, core_hi, (2, 2), "(- (+ 1.0 (* 0.002 i)) (* 0.001 j))")
    p.declare("e", core_lo, core_hi, (2, 2), "(+ 2.0 (* 0.001 (+ i j)))")
    p.declare("v", core_lo, core_hi, (2, 2), "(+ (+ 0.5 (* 0.003 i)) (* 0.001 j))")
    p.declare("gamma", core_lo, core_hi, (2, 2), 1.4)
    for t in ("t1", "t2", "t3", "t4", "t5", "t6"):
        p.declare(t, wlo, whi, (0, 0), 0.0)
    pt, s5, s3x, s3y = POINT, star(2), line(0), line(1)
    for it in range(iters):
        p.loop(wlo, whi, [("rho", s5, R), ("t1", pt, W)], {1: avg4(0)})
        p.loop(wlo, whi, [("e", s3x, R), ("t2", pt, W)], {1: mul(c(0.5), sub(r(0, 1, 0), r(0, -1, 0)))})
        p.loop(wlo, whi, [("v", s3y, R), ("t3", pt, W)], {1: mul(c(0.5), sub(r(0, 0, 1), r(0, 0, -1)))})
        p.loop(wlo, whi, [("t1", pt, R), ("t2", pt, R), ("t4", pt, W)], {2: add(r(0), r(1))})
        p.loop(wlo, whi, [("v", s5, R), ("t5", pt, W)], {1: avg4(0)})
        p.loop(wlo, whi, [("t3", pt, R), ("gamma", pt, R), ("e", pt, R), ("t6", pt, W)],
               {3: add(mul(r(0), r(1)), mul(c(0.001), r(2)))})
        p.loop(core_lo, core_hi, [("rho", pt, RW), ("t4", s3x, R)],
               {0: add(r(0), mul(c(0.01), sub(r(1, 1, 0), r(1, -1, 0))))})
        p.loop(core_lo, core_hi, [("e", pt, RW), ("t6", s3y, R)],
               {0: add(r(0), mul(c(0.01), sub(r(1, 0, 1), r(1, 0, -1))))})
        p.loop(core_lo, core_hi, [("v", pt, RW), ("t5", s5, R)],
               {0: add(mul(c(0.99), r(0)), mul(c(0.01), avg4(1)))})
        p.loop(wlo, whi, [("t4", pt, R), ("t5", pt, R), ("t2", pt, W)], {2: sub(r(0), r(1))})
        p.loop(wlo, whi, [("t1", pt, R), ("t2", pt, R), ("t3", pt, W)], {2: mn(r(0), r(1))})
        p.loop(core_lo, core_hi, [("rho", pt, RW), ("t2", pt, R)], {0: add(r(0), mul(c(0.001), r(1)))})
        p.loop(core_lo, core_hi, [("e", pt, RW), ("t3", pt, R)], {0: add(r(0), mul(c(0.002), r(1)))})
        p.loop(core_lo, core_hi, [("v", pt, RW), ("t3", s3x, R)],
               {0: add(r(0), mul(c(0.005), add(r(1, -1, 0), r(1, 1, 0))))})
        if (it + 1) % 10 == 0:
            p.loop(core_lo, core_hi, [("rho", pt, R), ("e", pt, R), ("v", pt, R), ("gamma", pt, R)],
                   None, ("SUM", add(add(r(0), r(1)), add(r(2), r(3))), "fieldsum"))
        if it == 1:
            p.flush()
            if cyclic:
                p.cyclic(True)
        if span > 0 and (it + 1) % span == 0:
            p.flush()
    p.finish()
    return p.to_dict()


RK_ALPHA = (1.0 / 3.0, 0.5, 1.0)  # apps.cpp:172
RK_BETA = (0.0, -0.6, -0.85)      # apps.cpp:173


def rk3chain(nx, ny, iters, span=0, cyclic=False):  # apps.cpp:156-213
    p = Prog()
    sp = span if span > 0 else 1
    pad = 3 * sp - 1
    lo, hi = (-pad, -pad), (nx + pad, ny + pad)
    p.declare("w", lo, hi, (1, 1), "(- (+ 1.0 (* 0.0015 i)) (* 0.0005 j))")
    p.declare("r", lo, hi, (0, 0), 0.0)
    p.declare("k", lo, hi, (0, 0), 0.0)
    p.declare("b", lo, hi, (0, 0), "(+ 1.0 (* 0.0001 (+ i (* 2 j))))")
    p.declare("c2", lo, hi, (0, 0), 0.9)
    p.declare("d3", lo, hi, (0, 0), 0.05)
    if cyclic:
        p.cyclic(True)
    pt, s5 = POINT, star(2)
    done = 0
    while done < iters:
        steps = min(sp, iters - done)
        for tau in range(steps):
            for sigma in range(3):
                depth = 3 * (steps - 1 - tau) + (2 - sigma)
                rlo, rhi = (-depth, -depth), (nx + depth, ny + depth)
                p.loop(rlo, rhi, [("w", s5, R), ("b", pt, R), ("r", pt, W)],
                       {2: mul(star5(0), r(1))})
                if sigma == 0:
                    p.loop(rlo, rhi, [("r", pt, R), ("c2", pt, R), ("k", pt, W)], {2: mul(r(0), r(1))})
                else:
                    p.loop(rlo, rhi, [("r", pt, R), ("c2", pt, R), ("k", pt, RW)],
                           {2: add(mul(c(RK_BETA[sigma]), r(2)), mul(r(0), r(1)))})
                p.loop(rlo, rhi, [("w", pt, RW), ("k", pt, R), ("d3", pt, R)],
                       {0: add(r(0), mul(c(RK_ALPHA[sigma]), mul(r(1), r(2))))})
        done += steps
        p.flush()
    p.finish()
    return p.to_dict()


# ----------------------------------------------------------------- 3-D analogues (new)


def avg6(arg):
    """6-neighbour average, the 3-D analogue of avg4."""
    return mul(c(1.0 / 6.0), add(add(add(r(arg, -1, 0, 0), r(arg, 1, 0, 0)),
                                     add(r(arg, 0, -1, 0), r(arg, 0, 1, 0))),
                                 add(r(arg, 0, 0, -1), r(arg, 0, 0, 1))))


def star7(arg):
    """7-point star, the 3-D analogue of star5."""
    return mul(c(1.0 / 7.0), add(add(add(add(r(arg, -1, 0, 0), r(arg, 1, 0, 0)),
                                         add(r(arg, 0, -1, 0), r(arg, 0, 1, 0))),
                                     add(r(arg, 0, 0, -1), r(arg, 0, 0, 1))), r(arg, 0, 0, 0)))


def miniflow3d(nx, ny, nz, iters, span=0, cyclic=False):
    """CloverLeaf-3D-shaped chain: miniflow2d's 14 loops with x/y/z derivatives."""
    p = Prog()
    core_lo, core_hi = (0, 0, 0), (nx, ny, nz)
    wlo, whi = (-1, -1, -1), (nx + 1, ny + 1, nz + 1)
    p.declare("rho", core_lo, core_hi, (2, 2, 2), "(+ (- (+ 1.0 (* 0.002 i)) (* 0.001 j)) (* 0.0005 k))")
    p.declare("e", core_lo, core_hi, (2, 2, 2), "(+ 2.0 (* 0.001 (+ (+ i j) k)))")
    p.declare("v", core_lo, core_hi, (2, 2, 2), "(- (+ (+ 0.5 (* 0.003 i)) (* 0.001 j)) (* 0.002 k))")
    p.declare("gamma", core_lo, core_hi, (2, 2, 2), 1.4)
    for t in ("t1", "t2", "t3", "t4", "t5", "t6"):
        p.declare(t, wlo, whi, (0, 0, 0), 0.0)
    pt, s7, s3x, s3y, s3z = POINT, star(3), line(0), line(1), line(2)
    for it in range(iters):
        p.loop(wlo, whi, [("rho", s7, R), ("t1", pt, W)], {1: avg6(0)})
        p.loop(wlo, whi, [("e", s3x, R), ("t2", pt, W)], {1: mul(c(0.5), sub(r(0, 1, 0, 0), r(0, -1, 0, 0)))})
        p.loop(wlo, whi, [("v", s3y, R), ("t3", pt, W)], {1: mul(c(0.5), sub(r(0, 0, 1, 0), r(0, 0, -1, 0)))})
        p.loop(wlo, whi, [("t1", pt, R), ("t2", pt, R), ("t4", pt, W)], {2: add(r(0), r(1))})
        p.loop(wlo, whi, [("v", s7, R), ("t5", pt, W)], {1: avg6(0)})
        p.loop(wlo, whi, [("t3", pt, R), ("gamma", pt, R), ("e", pt, R), ("t6", pt, W)],
               {3: add(mul(r(0), r(1)), mul(c(0.001), r(2)))})
        p.loop(core_lo, core_hi, [("rho", pt, RW), ("t4", s3x, R)],
               {0: add(r(0), mul(c(0.01), sub(r(1, 1, 0, 0), r(1, -1, 0, 0))))})
        p.loop(core_lo, core_hi, [("e", pt, RW), ("t6", s3z, R)],
               {0: add(r(0), mul(c(0.01), sub(r(1, 0, 0, 1), r(1, 0, 0, -1))))})
        p.loop(core_lo, core_hi, [("v", pt, RW), ("t5", s7, R)],
               {0: add(mul(c(0.99), r(0)), mul(c(0.01), avg6(1)))})
        p.loop(wlo, whi, [("t4", pt, R), ("t5", pt, R), ("t2", pt, W)], {2: sub(r(0), r(1))})
        p.loop(wlo, whi, [("t1", pt, R), ("t2", pt, R), ("t3", pt, W)], {2: mn(r(0), r(1))})
        p.loop(core_lo, core_hi, [("rho", pt, RW), ("t2", pt, R)], {0: add(r(0), mul(c(0.001), r(1)))})
        p.loop(core_lo, core_hi, [("e", pt, RW), ("t3", pt, R)], {0: add(r(0), mul(c(0.002), r(1)))})
        p.loop(core_lo, core_hi, [("v", pt, RW), ("t3", s3y, R)],
               {0: add(r(0), mul(c(0.005), add(r(1, 0, -1, 0), r(1, 0, 1, 0))))})
        if (it + 1) % 10 == 0:
            p.loop(core_lo, core_hi, [("rho", pt, R), ("e", pt, R), ("v", pt, R), ("gamma", pt, R)],
                   None, ("SUM", add(add(r(0), r(1)), add(r(2), r(3))), "fieldsum"))
        if it == 1:
            p.flush()
            if cyclic:
                p.cyclic(True)
        if span > 0 and (it + 1) % span == 0:
            p.flush()
    p.finish()
    return p.to_dict()


def rk3chain3d(nx, ny, nz, iters, span=0, cyclic=False):
    """OpenSBLI-TGV-shaped chain: rk3chain's three-stage low-storage scheme in 3-D."""
    p = Prog()
    sp = span if span > 0 else 1
    pad = 3 * sp - 1
    lo, hi = (-pad, -pad, -pad), (nx + pad, ny + pad, nz + pad)
    p.declare("w", lo, hi, (1, 1, 1), "(+ (- (+ 1.0 (* 0.0015 i)) (* 0.0005 j)) (* 0.00025 k))")
    p.declare("r", lo, hi, (0, 0, 0), 0.0)
    p.declare("k", lo, hi, (0, 0, 0), 0.0)
    p.declare("b", lo, hi, (0, 0, 0), "(+ 1.0 (* 0.0001 (+ (+ i (* 2 j)) (* 3 k))))")
    p.declare("c2", lo, hi, (0, 0, 0), 0.9)
    p.declare("d3", lo, hi, (0, 0, 0), 0.05)
    if cyclic:
        p.cyclic(True)
    pt, s7 = POINT, star(3)
    done = 0
    while done < iters:
        steps = min(sp, iters - done)
        for tau in range(steps):
            for sigma in range(3):
                depth = 3 * (steps - 1 - tau) + (2 - sigma)
                rlo, rhi = (-depth,) * 3, (nx + depth, ny + depth, nz + depth)
                p.loop(rlo, rhi, [("w", s7, R), ("b", pt, R), ("r", pt, W)], {2: mul(star7(0), r(1))})
                if sigma == 0:
                    p.loop(rlo, rhi, [("r", pt, R), ("c2", pt, R), ("k", pt, W)], {2: mul(r(0), r(1))})
                else:
                    p.loop(rlo, rhi, [("r", pt, R), ("c2", pt, R), ("k", pt, RW)],
                           {2: add(mul(c(RK_BETA[sigma]), r(2)), mul(r(0), r(1)))})
                p.loop(rlo, rhi, [("w", pt, RW), ("k", pt, R), ("d3", pt, R)],
                       {0: add(r(0), mul(c(RK_ALPHA[sigma]), mul(r(1), r(2))))})
        done += steps
        p.flush()
    p.finish()
    return p.to_dict()


APPS = {"heat2d": heat2d, "miniflow2d": miniflow2d, "rk3chain": rk3chain,
        "miniflow3d": miniflow3d, "rk3chain3d": rk3chain3d}


def app_program(name, nx, ny, nz=0, iters=10, span=0, cyclic=False):
    if name in ("miniflow3d", "rk3chain3d"):
        return APPS[name](nx, ny, nz or nx, iters, span, cyclic)
    return APPS[name](nx, ny, iters, span, cyclic)


# ----------------------------------------------------------------- random chains


def _rand_stencil(rng, ndim, max_extent):  # support.hpp:31-43
    s = [(0, 0, 0)]
    for _ in range(rng.randint(1, 5)):
        p = [0, 0, 0]
        for d in range(ndim):
            p[d] = rng.randint(-max_extent, max_extent)
        if tuple(p) not in s:
            s.append(tuple(p))
    return s


def _rand_expr(rng, reads, depth, ops):  # support.hpp:45-64 (+ divide)
    roll = rng.randint(0, 9)
    if depth <= 0 or roll < 4 or not reads:
        if reads and roll % 2 == 0:
            arg, st = reads[rng.randrange(len(reads))]
            o = st[rng.randrange(len(st))]
            return r(arg, *o)
        return c(round(rng.uniform(-2.0, 2.0), 6) if rng.random() < 0.5 else rng.uniform(-2.0, 2.0))
    op = ops[rng.randrange(len(ops))]
    return op(_rand_expr(rng, reads, depth - 1, ops), _rand_expr(rng, reads, depth - 1, ops))


def random_program(seed, max_loops=8, max_datasets=4, max_extent=2, min_size=8, max_size=24,
                   reductions=True, allow_3d=True, divide=True, flushes=False, max_3d=10, force_ndim=0):
    """A random validated-by-construction chain, support.hpp:66-138's distribution."""
    rng = random.Random(seed)
    roll = rng.randint(1, 6 if allow_3d else 4)
    ndim = 1 if roll <= 2 else 2 if roll <= 5 else 3
    if force_ndim:  # (consumes the same random draw, so other seeds' programs are unchanged)
        ndim = force_ndim
    dims = [1, 1, 1]
    for d in range(ndim):
        dims[d] = min(rng.randint(min_size, max_size), max_3d) if ndim == 3 else rng.randint(min_size, max_size)
    p = Prog()
    nds = rng.randint(1, max_datasets)
    names = [f"d{i}" for i in range(nds)]
    for nm in names:
        a, b, cc = (rng.uniform(-0.1, 0.1) for _ in range(3))
        fill = f"(+ (+ (+ 1.0 (* {_num(a)} i)) (* {_num(b)} j)) (* {_num(cc)} k))"
        p.declare(nm, [0] * ndim, dims[:ndim], [max_extent] * ndim, fill)
    ops = [add, sub, mul, mn, mx, add] + ([div] if divide else [])
    red_ops = ["SUM", "SUM", "MIN", "MAX"]
    for j in range(rng.randint(1, max_loops)):
        lo, hi = [0, 0, 0], [1, 1, 1]
        for d in range(ndim):
            lo[d] = rng.randint(0, dims[d] - 2)
            hi[d] = rng.randint(lo[d] + 1, dims[d])
        dw = rng.randrange(nds)
        rw = rng.randint(0, 9) < 3
        args = [(names[dw], POINT, RW if rw else W)]
        for _ in range(rng.randint(0, 2)):
            dr = rng.randrange(nds)
            if dr == dw or any(a[0] == names[dr] for a in args):
                continue
            args.append((names[dr], _rand_stencil(rng, ndim, max_extent), R))
        reads = [(i, a[1]) for i, a in enumerate(args) if a[2] != W]
        red = None
        if reductions and rng.randint(0, 9) < 2:
            red = (red_ops[rng.randrange(4)], _rand_expr(rng, reads, 2, ops), f"red{j}")
        p.loop(lo[:ndim], hi[:ndim], args, {0: _rand_expr(rng, reads, 3, ops)}, red)
        if flushes and rng.randint(0, 9) == 0:
            p.flush()
    p.finish()
    return p.to_dict()
