"""ORACLE — TEST INFRASTRUCTURE ONLY.

A CPU (numpy) restatement of the reference's out-of-core loop-chain path
(/root/reference/proj, "oocstencil"). Only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline leg may import this module, and only as the checker:
the product (paper_1709_02125_b200) never calls it and has no CPU fallback.

Parity pinning: this restatement is checked against golden vectors produced by
running the unmodified reference library (oracle/_ref/libooc_ref.so, built by
oracle/ref/Makefile from the reference sources) — see tests/golden/ and
tests/test_oracle_golden.py — and against the reference's own known-answer
tests (proj/tests/test_tiler.cpp:52-367, test_mesh_core.cpp:66-117).

Every function cites the reference file:line it restates. Arithmetic is IEEE
binary64 elementwise numpy (add/sub/mul/div correctly rounded, no FMA), the
same operations in the same order as the reference's tape interpreter
(proj/src/kernel_exec.cpp:46-88), so field results are bit-exact.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

I64_MIN = -(2 ** 63)
I64_MAX = 2 ** 63 - 1

# --------------------------------------------------------------------------
# Extent: half-open boxes of rank 1..3 (proj/include/ooc/extent.hpp:14-138)
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class Ext:
    ndim: int
    lo: Tuple[int, int, int]
    hi: Tuple[int, int, int]

    @staticmethod
    def make(ndim, lo, hi):  # extent.hpp:19-29
        lo = list(lo) + [0] * (3 - len(lo))
        hi = list(hi) + [1] * (3 - len(hi))
        for d in range(ndim, 3):
            lo[d], hi[d] = 0, 1
        return Ext(ndim, tuple(int(x) for x in lo), tuple(int(x) for x in hi))

    @staticmethod
    def none(ndim):  # extent.hpp:39
        return Ext.make(ndim, (0, 0, 0), (0, 0, 0))

    def empty(self):  # extent.hpp:41-45
        return any(self.lo[d] >= self.hi[d] for d in range(self.ndim))

    def length(self, d):
        return self.hi[d] - self.lo[d]

    def size(self):  # extent.hpp:49-54
        if self.empty():
            return 0
        n = 1
        for d in range(3):
            n *= self.hi[d] - self.lo[d]
        return n

    def contains(self, o: "Ext"):  # extent.hpp:62-67
        if o.empty():
            return True
        return all(o.lo[d] >= self.lo[d] and o.hi[d] <= self.hi[d] for d in range(3))

    def intersect(self, o: "Ext"):  # extent.hpp:69-78
        lo = tuple(max(self.lo[d], o.lo[d]) for d in range(3))
        hi = tuple(min(self.hi[d], o.hi[d]) for d in range(3))
        for d in range(self.ndim):
            if lo[d] >= hi[d]:
                return Ext.none(self.ndim)
        return Ext(self.ndim, lo, hi)

    def hull(self, o: "Ext"):  # extent.hpp:81-90
        if self.empty():
            return o
        if o.empty():
            return self
        return Ext(self.ndim, tuple(min(self.lo[d], o.lo[d]) for d in range(3)),
                   tuple(max(self.hi[d], o.hi[d]) for d in range(3)))

    def expand(self, lo_off, hi_off):  # extent.hpp:93-100
        lo, hi = list(self.lo), list(self.hi)
        for d in range(self.ndim):
            lo[d] += lo_off[d]
            hi[d] += hi_off[d]
        return Ext(self.ndim, tuple(lo), tuple(hi))

    def with_dim(self, d, l, h):  # extent.hpp:103-108
        lo, hi = list(self.lo), list(self.hi)
        lo[d], hi[d] = int(l), int(h)
        return Ext(self.ndim, tuple(lo), tuple(hi))

    def as_list(self):
        return [self.ndim, *self.lo, *self.hi]

    def shape(self):
        return tuple(self.hi[d] - self.lo[d] for d in range(3))


def stencil_extents(offsets):  # stencil.hpp:55-64
    if not offsets:
        raise ValidationError("stencil has no offsets")
    lo = [min(o[d] for o in offsets) for d in range(3)]
    hi = [max(o[d] for o in offsets) for d in range(3)]
    return tuple(lo), tuple(hi)


# --------------------------------------------------------------------------
# Errors (proj/include/ooc/errors.hpp:9-47)
# --------------------------------------------------------------------------


class ValidationError(Exception):
    pass


class StaleDataError(Exception):
    def __init__(self, name, chain):
        super().__init__(f"stale data: dataset '{name}' was discarded by chain {chain}")
        self.dataset, self.chain = name, chain


class InfeasibleError(Exception):
    def __init__(self, min_bytes, budget):
        super().__init__(f"infeasible tiling: minimum achievable 3-slot size is {min_bytes} "
                         f"bytes, budget is {budget} bytes")
        self.min_achievable_bytes = min_bytes


class CapacityError(Exception):
    def __init__(self, required, capacity):
        super().__init__(f"device capacity exceeded: {required} > {capacity}")
        self.required_bytes = required


# --------------------------------------------------------------------------
# Expressions: prefix parse + postfix tape (proj/src/expr.cpp:13-23, 73-147)
# --------------------------------------------------------------------------

BINOPS = {"+": "add", "-": "sub", "*": "mul", "/": "div", "min": "min", "max": "max"}


def _tokens(text):
    out, i, n = [], 0, len(text)
    while i < n:
        c = text[i]
        if c.isspace():
            i += 1
        elif c in "()":
            out.append(c)
            i += 1
        else:
            j = i
            while j < n and not text[j].isspace() and text[j] not in "()":
                j += 1
            out.append(text[i:j])
            i = j
    return out


def parse_prefix(text: str, allow_coords=False):
    """expr.cpp:73-123 — returns a nested tuple tree."""
    toks = _tokens(text)
    pos = [0]

    def nxt():
        if pos[0] >= len(toks):
            raise ValidationError("unexpected end of expression: " + text)
        t = toks[pos[0]]
        pos[0] += 1
        return t

    def rec():
        tok = nxt()
        if tok == ")":
            raise ValidationError("unexpected ')' in expression")
        if tok != "(":
            if allow_coords and tok in ("i", "j", "k"):
                return ("coord", "ijk".index(tok))
            try:
                return ("const", float(tok))
            except ValueError:
                raise ValidationError(f"unrecognised token '{tok}' in expression")
        head = nxt()
        if head == "r":
            arg = int(nxt())
            off = [0, 0, 0]
            d = 0
            while toks[pos[0]] != ")":
                off[d] = int(nxt())
                d += 1
            nxt()
            return ("read", arg, tuple(off))
        if head not in BINOPS:
            raise ValidationError(f"unknown operator '{head}' in expression")
        lhs = rec()
        rhs = rec()
        if nxt() != ")":
            raise ValidationError(f"operator '{head}' takes exactly two operands")
        return (BINOPS[head], lhs, rhs)

    tree = rec()
    if pos[0] != len(toks):
        raise ValidationError("trailing tokens after expression: " + text)
    return tree


def compile_tape(tree):
    """Postfix tape + max stack (expr.cpp:13-23, 134-140)."""
    tape = []
    maxd = [0]

    def rec(e, depth):
        if e[0] in ("add", "sub", "mul", "div", "min", "max"):
            rec(e[1], depth)
            rec(e[2], depth + 1)
            tape.append((e[0],))
        else:
            tape.append(e)
            maxd[0] = max(maxd[0], depth + 1)

    rec(tree, 0)
    return tape, maxd[0]


def tree_reads(tree):
    if tree[0] == "read":
        yield tree
    elif tree[0] in ("add", "sub", "mul", "div", "min", "max"):
        yield from tree_reads(tree[1])
        yield from tree_reads(tree[2])


def tree_has_coord(tree):
    if tree[0] == "coord":
        return True
    if tree[0] in ("add", "sub", "mul", "div", "min", "max"):
        return tree_has_coord(tree[1]) or tree_has_coord(tree[2])
    return False


def eval_tape(tape, load):
    """Vectorised restatement of eval() (kernel_exec.cpp:46-88): identical op
    order; std::min(a,b) = (b<a)?b:a, std::max(a,b) = (a<b)?b:a."""
    st = []
    with np.errstate(all="ignore"):
        for ins in tape:
            op = ins[0]
            if op == "const":
                st.append(np.float64(ins[1]))
            elif op in ("read", "coord"):
                st.append(load(ins))
            else:
                b = st.pop()
                a = st.pop()
                if op == "add":
                    st.append(a + b)
                elif op == "sub":
                    st.append(a - b)
                elif op == "mul":
                    st.append(a * b)
                elif op == "div":
                    st.append(a / b)
                elif op == "min":
                    st.append(np.where(b < a, b, a))
                else:
                    st.append(np.where(a < b, b, a))
    return st[0]


# --------------------------------------------------------------------------
# Datasets, loops, validation (dataset.cpp:5-38, loop.cpp:32-105, loop.hpp:21-115)
# --------------------------------------------------------------------------

READ, WRITE, RW = "READ", "WRITE", "READ_WRITE"


def reads(mode):
    return mode != WRITE


def writes(mode):
    return mode != READ


@dataclass
class Dataset:
    name: str
    core: Ext
    halo: Tuple[int, int, int]
    elem_bytes: int
    host: np.ndarray  # shaped by alloc().shape(), always 3-D
    host_stale: bool = False
    stale_chain: int = -1
    stale_region: Optional[Ext] = None
    ever_written: bool = False

    def alloc(self):  # dataset.hpp:36-43
        lo = list(self.core.lo)
        hi = list(self.core.hi)
        for d in range(self.core.ndim):
            lo[d] -= self.halo[d]
            hi[d] += self.halo[d]
        return Ext(self.core.ndim, tuple(lo), tuple(hi))


@dataclass
class Arg:
    dataset: int
    offsets: List[Tuple[int, int, int]]
    mode: str


@dataclass
class Loop:
    range: Ext
    args: List[Arg]
    writes: List[Tuple[int, tuple]]  # (arg, tree)
    reduce_op: Optional[str] = None  # SUM / MIN / MAX
    reduce_tree: Optional[tuple] = None
    reduce_name: str = ""
    id: int = -1
    write_tapes: list = field(default_factory=list)
    reduce_tape: list = field(default_factory=list)

    def writes_dataset(self, d):
        return any(a.dataset == d and writes(a.mode) for a in self.args)


def loop_bytes_per_point(mesh, loop):  # loop.hpp:83-88
    return sum(mesh[a.dataset].elem_bytes * (2 if a.mode == RW else 1) for a in loop.args)


def loop_metric_bytes(mesh, loop):  # metrics.cpp:10-12
    return loop.range.size() * loop_bytes_per_point(mesh, loop)


def validate_loop(mesh: List[Dataset], loop: Loop):  # loop.cpp:32-105
    if loop.range.empty():
        raise ValidationError("loop has an empty iteration range")
    if not loop.args and not loop.writes and loop.reduce_op is None:
        raise ValidationError("loop has no arguments and no reduction")
    for a in loop.args:
        if a.dataset < 0 or a.dataset >= len(mesh):
            raise ValidationError("loop argument names an unknown dataset")
        if not a.offsets:
            raise ValidationError("loop argument has an empty stencil")
        ds = mesh[a.dataset]
        if loop.range.ndim != ds.core.ndim:
            raise ValidationError(f"loop rank does not match dataset '{ds.name}'")
        for off in a.offsets:
            for d in range(ds.core.ndim, 3):
                if off[d] != 0:
                    raise ValidationError("stencil offset uses a dimension beyond the rank")
        if writes(a.mode):
            if not (len(a.offsets) == 1 and tuple(a.offsets[0]) == (0, 0, 0)):
                raise ValidationError(f"write access to '{ds.name}' must use the single "
                                      "zero-offset stencil")
            if not ds.core.contains(loop.range):
                raise ValidationError(f"loop range exceeds the core of written dataset '{ds.name}'")
        if reads(a.mode):
            lo, hi = stencil_extents(a.offsets)
            if not ds.alloc().contains(loop.range.expand(lo, hi)):
                raise ValidationError(f"loop reads beyond the allocation of '{ds.name}'")
    for i, a in enumerate(loop.args):
        if not writes(a.mode):
            continue
        for k, b in enumerate(loop.args):
            if k != i and b.dataset == a.dataset:
                raise ValidationError(f"dataset '{mesh[a.dataset].name}' is written and appears "
                                      "in another argument of the same loop")
    written = [False] * len(loop.args)

    def check_reads(tree):
        if tree_has_coord(tree):
            raise ValidationError("coordinate terms are only valid in fill expressions")
        for r in tree_reads(tree):
            arg = r[1]
            if arg < 0 or arg >= len(loop.args):
                raise ValidationError(f"reads argument {arg} which does not exist")
            a = loop.args[arg]
            if not reads(a.mode):
                raise ValidationError(f"reads argument {arg} declared WRITE")
            if tuple(r[2]) not in [tuple(o) for o in a.offsets]:
                raise ValidationError("read offset not in the declared stencil")

    for arg, tree in loop.writes:
        if arg < 0 or arg >= len(loop.args):
            raise ValidationError(f"kernel writes argument {arg} which does not exist")
        if not writes(loop.args[arg].mode):
            raise ValidationError(f"kernel writes argument {arg} declared READ")
        if written[arg]:
            raise ValidationError(f"kernel writes argument {arg} twice")
        written[arg] = True
        check_reads(tree)
    for i, a in enumerate(loop.args):
        if writes(a.mode) and not written[i]:
            raise ValidationError(f"argument {i} is declared writable but the kernel never writes it")
    if loop.reduce_op is not None:
        if loop.reduce_tree is None:
            raise ValidationError("reduction without an expression")
        if not loop.reduce_name:
            raise ValidationError("reduction without a name")
        check_reads(loop.reduce_tree)
    loop.write_tapes = [compile_tape(t)[0] for _, t in loop.writes]
    loop.reduce_tape = compile_tape(loop.reduce_tree)[0] if loop.reduce_op else []


# --------------------------------------------------------------------------
# Kernel application (kernel_exec.cpp:133-198) and reductions (loop.hpp:92-115)
# --------------------------------------------------------------------------


def reduce_identity(op):
    return {"SUM": 0.0, "MIN": math.inf, "MAX": -math.inf}.get(op, 0.0)


def reduce_fold(op, acc, vals):
    """Strictly sequential row-major fold (kernel_exec.cpp:193-197)."""
    vals = np.ascontiguousarray(vals, dtype=np.float64).ravel()
    if vals.size == 0:
        return acc
    if op == "SUM":
        seq = np.empty(vals.size + 1)
        seq[0] = acc
        seq[1:] = vals
        return float(np.add.accumulate(seq)[-1])  # left fold, no pairwise summation
    # std::min(acc, v) = (v < acc) ? v : acc ; std::max(acc, v) = (acc < v) ? v : acc
    if math.isnan(acc):
        return acc
    vals = vals[~np.isnan(vals)]
    seq = np.concatenate([[acc], vals])
    m = seq.min() if op == "MIN" else seq.max()
    return float(seq[int(np.argmax(seq == m))])  # first extremum wins ties (e.g. +0/-0)


def apply_loop(mesh, loop: Loop, rng: Ext, acc: Optional[float] = None):
    """Whole-allocation views (reference.cpp:7-25 → apply_loop). Writes land after
    every tape of the point is evaluated (kernel_exec.cpp:173-179)."""
    if rng.empty():
        return acc

    def load(ins):
        _, arg, off = ins
        ds = mesh[loop.args[arg].dataset]
        box = ds.alloc()
        sl = tuple(slice(rng.lo[d] + off[d] - box.lo[d], rng.hi[d] + off[d] - box.lo[d])
                   for d in range(3))
        return ds.host[sl]

    outs = [np.broadcast_to(eval_tape(t, load), rng.shape()).copy() for t in loop.write_tapes]
    red = None
    if loop.reduce_op is not None and acc is not None:
        red = np.broadcast_to(eval_tape(loop.reduce_tape, load), rng.shape()).copy()
    for (arg, _), val in zip(loop.writes, outs):
        ds = mesh[loop.args[arg].dataset]
        box = ds.alloc()
        sl = tuple(slice(rng.lo[d] - box.lo[d], rng.hi[d] - box.lo[d]) for d in range(3))
        ds.host[sl] = val
    if red is not None:
        acc = reduce_fold(loop.reduce_op, acc, red)
    return acc


# --------------------------------------------------------------------------
# Planner (tiler.cpp:18-136, 138-294, 383-433)
# --------------------------------------------------------------------------


def access_extent(loop: Loop, d, dim):  # tiler.cpp:25-43
    rd = wr = False
    rlo = rhi = 0
    for a in loop.args:
        if a.dataset != d:
            continue
        if writes(a.mode):
            wr = True
        if reads(a.mode):
            lo, hi = stencil_extents(a.offsets)
            if not rd:
                rlo, rhi = lo[dim], hi[dim]
            else:
                rlo, rhi = min(rlo, lo[dim]), max(rhi, hi[dim])
            rd = True
    return rd, wr, rlo, rhi


def chain_datasets(mesh, loops):  # tiler.cpp:45-53
    used = sorted({a.dataset for l in loops for a in l.args})
    return used


def union_is_box(a: Ext, b: Ext):  # tiler.cpp:56-66
    if a.contains(b) or b.contains(a):
        return True
    odd = -1
    for d in range(3):
        if a.lo[d] == b.lo[d] and a.hi[d] == b.hi[d]:
            continue
        if odd >= 0:
            return False
        odd = d
    if odd < 0:
        return True
    return max(a.lo[odd], b.lo[odd]) <= min(a.hi[odd], b.hi[odd])


@dataclass
class TilePlan:
    tiled_dim: int
    tile_count: int
    nominal_ends: List[int]
    loop_ranges: List[Ext]
    ends: List[List[int]]
    warnings: List[str]

    def subrange(self, j, t):  # tiler.hpp:31-37
        start = self.loop_ranges[j].lo[self.tiled_dim] if t == 0 else self.ends[j][t - 1]
        end = self.ends[j][t]
        r = self.loop_ranges[j].with_dim(self.tiled_dim, start, end)
        if start >= end:
            return Ext.make(r.ndim, (0, 0, 0), (0, 0, 0))
        return r


def compute_tile_plan(mesh, loops: Sequence[Loop], tile_count, tiled_dim=0):  # tiler.cpp:70-136
    if not loops:
        raise ValidationError("cannot tile an empty chain")
    if tile_count < 1:
        raise ValidationError("tile count must be at least 1")
    ndim = loops[0].range.ndim
    if tiled_dim < 0 or tiled_dim >= ndim:
        raise ValidationError("tiled dimension out of range")
    lo = min(l.range.lo[tiled_dim] for l in loops)
    hi = max(l.range.hi[tiled_dim] for l in loops)
    extent = hi - lo
    warnings = []
    if tile_count > extent:
        warnings.append(f"tile count {tile_count} exceeds tiled extent {extent}; reduced")
        tile_count = extent
    nominal = [lo + ((t + 1) * extent) // tile_count for t in range(tile_count)]
    n = len(loops)
    ends = [[0] * tile_count for _ in range(n)]
    ae_cache = [{a.dataset: access_extent(l, a.dataset, tiled_dim) for a in l.args} for l in loops]
    nd = len(mesh)
    for t in range(tile_count):
        read_req = [I64_MIN] * nd
        write_req = [I64_MIN] * nd
        for j in range(n - 1, -1, -1):
            loop = loops[j]
            d = nominal[t]
            for a in loop.args:
                rd, wr, rlo, rhi = ae_cache[j][a.dataset]
                if writes(a.mode):
                    if read_req[a.dataset] != I64_MIN:
                        d = max(d, read_req[a.dataset])
                    if write_req[a.dataset] != I64_MIN:
                        d = max(d, write_req[a.dataset])
                if reads(a.mode) and write_req[a.dataset] != I64_MIN:
                    d = max(d, write_req[a.dataset] - rlo)
            d = min(max(d, loop.range.lo[tiled_dim]), loop.range.hi[tiled_dim])
            if t == tile_count - 1:
                d = loop.range.hi[tiled_dim]
            if t > 0:
                d = max(d, ends[j][t - 1])
            ends[j][t] = d
            for a in loop.args:
                rd, wr, rlo, rhi = ae_cache[j][a.dataset]
                if reads(a.mode):
                    read_req[a.dataset] = max(read_req[a.dataset], d + rhi)
                if writes(a.mode):
                    write_req[a.dataset] = max(write_req[a.dataset], d)
    return TilePlan(tiled_dim, tile_count, nominal, [l.range for l in loops], ends, warnings)


@dataclass
class PerDataset:
    accessed: bool = False
    written_any: bool = False
    write_first: bool = False
    full: list = field(default_factory=list)
    left_edge: list = field(default_factory=list)
    right_edge: list = field(default_factory=list)
    left_fp: list = field(default_factory=list)
    right_fp: list = field(default_factory=list)
    modified: list = field(default_factory=list)
    max_tile_bytes: int = 0


@dataclass
class Footprints:
    per_dataset: List[PerDataset]
    slot_bytes: int = 0


def compute_footprints(mesh, loops: Sequence[Loop], plan: TilePlan):  # tiler.cpp:138-294
    T, dim, n = plan.tile_count, plan.tiled_dim, len(loops)
    fp = Footprints([PerDataset() for _ in mesh])
    used = chain_datasets(mesh, loops)
    for d in used:
        pd = fp.per_dataset[d]
        pd.accessed = True
        alloc = mesh[d].alloc()
        empty = Ext.none(alloc.ndim)
        pd.full = [empty] * T
        pd.left_edge = [empty] * T
        pd.right_edge = [empty] * T
        pd.left_fp = [empty] * T
        pd.right_fp = [empty] * T
        pd.modified = [0] * T
        base = None
        for loop in loops:  # :159-180
            uses = False
            elo, ehi = [0, 0, 0], [0, 0, 0]
            for a in loop.args:
                if a.dataset != d:
                    continue
                uses = True
                if reads(a.mode):
                    slo, shi = stencil_extents(a.offsets)
                    for k in range(3):
                        elo[k] = min(elo[k], slo[k])
                        ehi[k] = max(ehi[k], shi[k])
            if not uses:
                continue
            reach = loop.range.expand(elo, ehi).intersect(alloc)
            base = reach if base is None else base.hull(reach)
        a_t = [I64_MAX] * T
        b_t = [I64_MIN] * T
        for t in range(T):  # :183-200
            for j, loop in enumerate(loops):
                rd, wr, rlo, rhi = access_extent(loop, d, dim)
                if not rd and not wr:
                    continue
                sub = plan.subrange(j, t)
                if sub.empty():
                    continue
                lo_ = min(0, rlo) if rd else 0
                hi_ = max(0, rhi) if rd else 0
                a_t[t] = min(a_t[t], sub.lo[dim] + lo_)
                b_t[t] = max(b_t[t], sub.hi[dim] + hi_)
                if wr:
                    pd.modified[t] = 1
            a_t[t] = max(a_t[t], alloc.lo[dim])
            b_t[t] = min(b_t[t], alloc.hi[dim])
        nonempty = lambda t: a_t[t] < b_t[t]
        prev = -1
        for t in range(T):  # :206-211
            if not nonempty(t):
                continue
            if prev >= 0:
                b_t[t] = max(b_t[t], b_t[prev])
            prev = t
        nxt = -1
        for t in range(T - 1, -1, -1):  # :212-217
            if not nonempty(t):
                continue
            if nxt >= 0:
                a_t[t] = min(a_t[t], a_t[nxt])
            nxt = t
        prev = -1
        for t in range(T):  # :220-229
            if not nonempty(t):
                continue
            if prev >= 0 and t > prev + 1 and a_t[t] < b_t[prev]:
                for g in range(prev + 1, t):
                    a_t[g] = a_t[t]
                    b_t[g] = b_t[prev]
            prev = t
        eb = mesh[d].elem_bytes
        for t in range(T):  # :231-236
            if a_t[t] >= b_t[t]:
                continue
            pd.full[t] = base.with_dim(dim, a_t[t], b_t[t])
            pd.max_tile_bytes = max(pd.max_tile_bytes, pd.full[t].size() * eb)
            if pd.modified[t]:
                pd.written_any = True
        for t in range(T):  # :237-251
            full = pd.full[t]
            if full.empty():
                continue
            if t > 0 and not pd.full[t - 1].empty():
                pd.left_edge[t] = full.intersect(pd.full[t - 1])
            if t + 1 < T and not pd.full[t + 1].empty():
                pd.right_edge[t] = full.intersect(pd.full[t + 1])
            pd.left_fp[t] = (full if pd.right_edge[t].empty()
                             else full.with_dim(dim, full.lo[dim], pd.right_edge[t].lo[dim]))
            pd.right_fp[t] = (full if pd.left_edge[t].empty()
                              else full.with_dim(dim, pd.left_edge[t].hi[dim], full.hi[dim]))
            if pd.left_fp[t].lo[dim] >= pd.left_fp[t].hi[dim]:
                pd.left_fp[t] = Ext.none(full.ndim)
            if pd.right_fp[t].lo[dim] >= pd.right_fp[t].hi[dim]:
                pd.right_fp[t] = Ext.none(full.ndim)
        fp.slot_bytes += pd.max_tile_bytes
    for d in used:  # :260-292 write-first qualification
        pd = fp.per_dataset[d]
        written = None
        exact, reads_prior = True, False
        for loop in loops:
            for a in loop.args:
                if a.dataset != d:
                    continue
                if reads(a.mode):
                    slo, shi = stencil_extents(a.offsets)
                    reach = loop.range.expand(slo, shi)
                    if written is None or not exact or not written.contains(reach):
                        reads_prior = True
                if writes(a.mode):
                    if written is None:
                        written = loop.range
                    elif written.contains(loop.range):
                        pass
                    elif union_is_box(written, loop.range):
                        written = written.hull(loop.range)
                    else:
                        written = written.hull(loop.range)
                        exact = False
        covered = written is not None and exact
        if covered:
            for t in range(T):
                if not pd.full[t].empty() and not written.contains(pd.full[t]):
                    covered = False
                    break
        pd.write_first = (not reads_prior) and covered
    return fp


def choose_tile_count(mesh, loops, budget, tiled_dim=0):  # tiler.cpp:383-402
    if budget <= 0:
        raise ValidationError("tile budget must be positive")
    lo = min(l.range.lo[tiled_dim] for l in loops)
    hi = max(l.range.hi[tiled_dim] for l in loops)
    min_seen = I64_MAX
    for T in range(1, hi - lo + 1):
        plan = compute_tile_plan(mesh, loops, T, tiled_dim)
        fp = compute_footprints(mesh, loops, plan)
        min_seen = min(min_seen, 3 * fp.slot_bytes)
        if 3 * fp.slot_bytes <= budget:
            return plan, fp
    raise InfeasibleError(min_seen, budget)


def chain_structural_key(mesh, loops):  # tiler.cpp:404-417
    parts = []
    for l in loops:
        s = f"L{l.range.ndim}" + "".join(f",{l.range.lo[d]},{l.range.hi[d]}" for d in range(3))
        for a in l.args:
            mode = {READ: 0, WRITE: 1, RW: 2}[a.mode]
            s += f";{a.dataset}:{mode}:" + "".join(f"{o[0]}.{o[1]}.{o[2]} " for o in a.offsets)
            s += "@" + repr(mesh[a.dataset].alloc().as_list())
        parts.append(s + "|")
    return "".join(parts)


def plan_json(mesh, plan: TilePlan, fp: Footprints):
    """Same schema as oracle/ref/ref_capi.cpp full_plan_json (golden fixtures)."""
    ds = []
    for d, pd in enumerate(fp.per_dataset):
        jd = {"name": mesh[d].name, "accessed": pd.accessed}
        if pd.accessed:
            jd.update(written_any=pd.written_any, write_first=pd.write_first,
                      max_tile_bytes=pd.max_tile_bytes, modified=list(pd.modified))
            for key in ("full", "left_edge", "right_edge", "left_fp", "right_fp"):
                jd[key] = [e.as_list() for e in getattr(pd, key)]
        ds.append(jd)
    return {"T": plan.tile_count, "tiled_dim": plan.tiled_dim, "nominal_ends": plan.nominal_ends,
            "ends": plan.ends, "warnings": len(plan.warnings), "slot_bytes": fp.slot_bytes,
            "datasets": ds}


# --------------------------------------------------------------------------
# Runtime: lazy queue, flush, executors (runtime.cpp:5-148, explicit_exec.cpp:55-281)
# --------------------------------------------------------------------------


class Runtime:
    """Observable restatement of ooc::Runtime for executors 'reference' and
    'explicit'. The explicit executor's observable effects are restated exactly:
    final host buffers (the three-slot data flow lands every chain value in the
    union of left footprints, tiler.cpp:237-251, which is what the reference's
    byte-conservation test proves — test_device_sim.cpp:228-263), per-(dataset,
    tile) audit bytes (explicit_exec.cpp:86-130, 173-243), cyclic discards and
    stale bookkeeping (explicit_exec.cpp:233-258), reductions folded in tile
    order == row-major order (explicit_exec.cpp:159-162)."""

    def __init__(self, executor="reference", tiles=0, capacity=16000000000, record=False,
                 prefetch=False):
        self.prefetch = prefetch
        self.staged = {}  # dataset -> region staged for the next chain (DeviceState::staged)
        self.executor = executor
        self.tiles = tiles
        self.capacity = capacity
        self.record = record
        self.mesh: List[Dataset] = []
        self.pending: List[Loop] = []
        self.cyclic = False
        self.next_loop_id = 0
        self.next_chain_id = 0
        self.flush_log = []
        self.chain_log = []
        self.audit = []
        self.reductions: Dict[str, float] = {}
        self.metric_bytes = 0
        self.uploaded = self.downloaded = self.d2d = 0
        self.tile_counts = []
        self.block_ndim = 0
        self._plans = {}

    # dataset.cpp:5-38
    def declare(self, name, core: Ext, halo, elem_bytes=8, fill=0.0):
        if any(d.name == name for d in self.mesh):
            raise ValidationError(f"duplicate dataset name '{name}'")
        if core.empty():
            raise ValidationError(f"dataset '{name}' has a zero-size core extent")
        if self.block_ndim == 0:
            self.block_ndim = core.ndim
        elif self.block_ndim != core.ndim:
            raise ValidationError(f"dataset '{name}' has rank {core.ndim} but its block has "
                                  f"rank {self.block_ndim}")
        halo = tuple(int(halo[d]) if d < core.ndim else 0 for d in range(3))
        if any(h < 0 for h in halo):
            raise ValidationError(f"dataset '{name}' has a negative halo depth")
        if elem_bytes <= 0:
            raise ValidationError(f"dataset '{name}' has non-positive elem_bytes")
        ds = Dataset(name, core, halo, elem_bytes, None, stale_region=Ext.none(core.ndim))
        a = ds.alloc()
        if isinstance(fill, str):
            tape, _ = compile_tape(parse_prefix(fill, allow_coords=True))
            grids = np.meshgrid(*[np.arange(a.lo[d], a.hi[d], dtype=np.int64) for d in range(3)],
                                indexing="ij")

            def load(ins):
                if ins[0] == "read":
                    raise ValidationError("fill expressions cannot read datasets")
                return grids[ins[1]].astype(np.float64)

            ds.host = np.broadcast_to(eval_tape(tape, load), a.shape()).astype(np.float64).copy()
        elif callable(fill):
            ds.host = np.asarray(fill(a), dtype=np.float64).reshape(a.shape()).copy()
        else:
            ds.host = np.full(a.shape(), float(fill))
        self.mesh.append(ds)
        return len(self.mesh) - 1

    def find(self, name):
        for i, d in enumerate(self.mesh):
            if d.name == name:
                return i
        return -1

    def enqueue_loop(self, loop: Loop):  # runtime.cpp:5-11
        validate_loop(self.mesh, loop)
        loop.id = self.next_loop_id
        self.next_loop_id += 1
        self.pending.append(loop)
        if loop.reduce_op is not None:
            self.flush("REDUCTION_FETCH")

    def fetch_dataset(self, d):  # runtime.cpp:13-19
        self.flush("DATA_FETCH")
        ds = self.mesh[d]
        if ds.host_stale:
            raise StaleDataError(ds.name, ds.stale_chain)
        self.staged.pop(d, None)  # returned data may change before the next chain (:17)
        return ds.host.copy()

    def fetch_reduction(self, name):  # runtime.cpp:21-26
        self.flush("DATA_FETCH")
        if name not in self.reductions:
            raise ValidationError(f"unknown reduction '{name}'")
        return self.reductions[name]

    def set_cyclic_flag(self, on):
        self.cyclic = bool(on)

    def finish(self):
        self.flush("PROGRAM_END")

    def flush(self, reason="EXPLICIT_FLUSH"):  # runtime.cpp:28-39
        if not self.pending:
            return
        loops, self.pending = self.pending, []
        cid = self.next_chain_id
        self.next_chain_id += 1
        self.flush_log.append((cid, reason, len(loops)))
        if self.record:
            self.chain_log.append(loops)
        self._execute(cid, loops)

    def plan_for(self, loops):  # runtime.cpp:41-62 (+ PlanCache, tiler.cpp:419-433)
        if self.tiles > 0:
            T = self.tiles
        else:
            plan, _ = choose_tile_count(self.mesh, loops, self.capacity)
            T = plan.tile_count
        key = (T, chain_structural_key(self.mesh, loops))
        if key not in self._plans:
            plan = compute_tile_plan(self.mesh, loops, T)
            self._plans[key] = (plan, compute_footprints(self.mesh, loops, plan))
        return self._plans[key]

    def _execute(self, cid, loops):  # runtime.cpp:64-148
        for l in loops:
            self.metric_bytes += loop_metric_bytes(self.mesh, l)
        if self.executor == "reference":
            for l in loops:
                for a in l.args:
                    if writes(a.mode):
                        self.mesh[a.dataset].ever_written = True
                acc = reduce_identity(l.reduce_op) if l.reduce_op else None
                acc = apply_loop(self.mesh, l, l.range, acc)
                if l.reduce_op:
                    self.reductions[l.reduce_name] = acc
            self.tile_counts.append(1)
            return
        plan, fp = self.plan_for(loops)
        self.tile_counts.append(plan.tile_count)
        for d, pd in enumerate(fp.per_dataset):  # runtime.cpp:98-105 stale-input guard
            if pd.accessed and self.mesh[d].host_stale and not pd.write_first:
                raise StaleDataError(self.mesh[d].name, self.mesh[d].stale_chain)
        if 3 * fp.slot_bytes > self.capacity:  # explicit_exec.cpp:61-62
            raise CapacityError(3 * fp.slot_bytes, self.capacity)
        self._run_explicit(cid, loops, plan, fp)

    def _run_explicit(self, cid, loops, plan: TilePlan, fp: Footprints):
        T = plan.tile_count
        used = [d for d, pd in enumerate(fp.per_dataset) if pd.accessed]
        audit = {}

        def row(d, t):
            return audit.setdefault((d, t), [d, t, 0, 0, 0])

        # uploads: tile-0 full footprint on q0, right footprints of t+1 on q1
        # (explicit_exec.cpp:174-186; write-first never travels up, :86)
        dim = plan.tiled_dim
        for d in used:
            pd = fp.per_dataset[d]
            eb = self.mesh[d].elem_bytes
            if pd.write_first:
                continue
            region = pd.full[0]
            if not region.empty():
                # tile-0 upload consumes a speculative stage when it only differs along
                # the tiled dimension (explicit_exec.cpp:135-157)
                st = self.staged.get(d)
                common = region.intersect(st) if st is not None else Ext.none(region.ndim)
                splits = not common.empty() and all(
                    k == dim or (common.lo[k] == region.lo[k] and common.hi[k] == region.hi[k])
                    for k in range(3))
                if splits:
                    if region.lo[dim] < common.lo[dim]:
                        row(d, 0)[2] += region.with_dim(dim, region.lo[dim], common.lo[dim]).size() * eb
                    if common.hi[dim] < region.hi[dim]:
                        row(d, 0)[2] += region.with_dim(dim, common.hi[dim], region.hi[dim]).size() * eb
                else:
                    row(d, 0)[2] += region.size() * eb
            for t in range(1, T):
                if not pd.right_fp[t].empty():
                    row(d, t)[2] += pd.right_fp[t].size() * eb
        self.staged = {}  # anything not consumed is for a chain that never came (:178)
        if self.prefetch:  # stage this chain's first tile for the next chain (:188-204, 260-271)
            for d in used:
                pd = fp.per_dataset[d]
                if pd.write_first or pd.full[0].empty():
                    continue
                row(d, T)[2] += pd.full[0].size() * self.mesh[d].elem_bytes
                self.staged[d] = pd.full[0]
        # device-to-device edge carry (:230-231)
        for t in range(T - 1):
            for d in used:
                e = fp.per_dataset[d].right_edge[t]
                if not e.empty():
                    row(d, t + 1)[4] += e.size() * self.mesh[d].elem_bytes
        # pre-chain host snapshot of datasets the cyclic mode will discard
        discard = [d for d in used if self.cyclic and fp.per_dataset[d].write_first
                   and fp.per_dataset[d].written_any]
        saved = {d: self.mesh[d].host.copy() for d in discard}
        # computation: tile-ordered execution equals loop-ordered execution for a
        # plan passing the dependency oracle (tiler.cpp:296-381); reductions fold
        # tile sub-ranges in tile order == row-major order (explicit_exec.cpp:159-162)
        for l in loops:
            for a in l.args:
                if writes(a.mode):
                    self.mesh[a.dataset].ever_written = True
            acc = reduce_identity(l.reduce_op) if l.reduce_op else None
            acc = apply_loop(self.mesh, l, l.range, acc)
            if l.reduce_op:
                self.reductions[l.reduce_name] = acc
        # downloads (:233-242) and staleness (:245-258)
        for d in used:
            pd = fp.per_dataset[d]
            ds = self.mesh[d]
            if not pd.written_any:
                continue
            down_hull = Ext.none(ds.alloc().ndim)
            skip_hull = Ext.none(ds.alloc().ndim)
            for t in range(T):
                if self.cyclic and pd.write_first:
                    skip_hull = skip_hull.hull(pd.left_fp[t])
                    continue
                if not pd.left_fp[t].empty():
                    row(d, t)[3] += pd.left_fp[t].size() * ds.elem_bytes
                down_hull = down_hull.hull(pd.left_fp[t])
            if not skip_hull.empty():
                ds.host[...] = saved[d]
                ds.stale_region = ds.stale_region.hull(skip_hull) if ds.host_stale else skip_hull
                ds.host_stale = True
                ds.stale_chain = cid
            elif ds.host_stale and not down_hull.empty() and down_hull.contains(ds.stale_region):
                ds.host_stale = False
                ds.stale_chain = -1
                ds.stale_region = Ext.none(ds.alloc().ndim)
        for k in sorted(audit):
            r = audit[k]
            self.audit.append(tuple(r))
            self.uploaded += r[2]
            self.downloaded += r[3]
            self.d2d += r[4]


# --------------------------------------------------------------------------
# Programs: the reference chain-file JSON (chain_file.cpp:58-162) + "ops"
# --------------------------------------------------------------------------


def ext_from_json(j):  # chain_file.cpp:13-26
    lo, hi = j["lo"], j["hi"]
    if len(lo) != len(hi) or not lo or len(lo) > 3:
        raise ValidationError("extent arrays must have matching rank 1..3")
    return Ext.make(len(lo), lo, hi)


def loop_from_json(rt: Runtime, stencils, jl) -> Loop:  # chain_file.cpp:134-159
    args = []
    for ja in jl["args"]:
        d = rt.find(ja["dataset"])
        if d < 0:
            raise ValidationError(f"loop argument names unknown dataset '{ja['dataset']}'")
        args.append(Arg(d, stencils[ja["stencil"]], ja["mode"]))
    k = jl.get("kernel", {})
    ws = [(int(a), parse_prefix(e)) for a, e in sorted(k.get("writes", {}).items())]
    loop = Loop(ext_from_json(jl["range"]), args, ws)
    if "reduction" in k:
        r = k["reduction"]
        loop.reduce_op = r["op"]
        loop.reduce_tree = parse_prefix(r["expr"])
        loop.reduce_name = r["name"]
    return loop


def load_program(rt: Runtime, prog):
    """Declare datasets, then replay ops (loops / flush / cyclic / finish)."""
    if isinstance(prog, str):
        prog = json.loads(prog)
    for jd in prog.get("datasets", []):
        core = ext_from_json(jd["core"])
        h = jd.get("halo", 0)
        halo = [h] * core.ndim if isinstance(h, int) else list(h)
        rt.declare(jd["name"], core, halo + [0] * (3 - len(halo)), jd.get("elem_bytes", 8),
                   jd.get("fill", 0.0))
    stencils = {"point": [(0, 0, 0)]}
    for js in prog.get("stencils", []):
        stencils[js["name"]] = [tuple(list(o) + [0] * (3 - len(o))) for o in js["offsets"]]
    ops = prog.get("ops")
    if ops is None:
        ops = [dict(l, op="loop") for l in prog.get("loops", [])]
    for op in ops:
        kind = op["op"]
        if kind == "loop":
            rt.enqueue_loop(loop_from_json(rt, stencils, op))
        elif kind == "flush":
            rt.flush()
        elif kind == "finish":
            rt.finish()
        elif kind == "cyclic":
            rt.set_cyclic_flag(op.get("on", True))
        else:
            raise ValidationError(f"unknown program op '{kind}'")
    return rt


# --------------------------------------------------------------------------
# Checksums shared with the golden generator
# --------------------------------------------------------------------------


def checksum(arr) -> str:
    """Order-sensitive 64-bit mix of the raw IEEE bits (used by tests/golden)."""
    x = np.ascontiguousarray(arr, dtype=np.float64).ravel().view(np.uint64)
    with np.errstate(over="ignore"):
        i = np.arange(x.size, dtype=np.uint64)
        k = (i * np.uint64(0x9E3779B97F4A7C15) + np.uint64(0x632BE59BD9B4E019)) | np.uint64(1)
        m = (x ^ (x >> np.uint64(29))) * k
        h = np.bitwise_xor.reduce(m ^ (m >> np.uint64(32))) if x.size else np.uint64(0)
        s = np.add.reduce(m, dtype=np.uint64) if x.size else np.uint64(0)
    return f"{int(h):016x}{int(s):016x}"
