"""ooc-b200: a B200-native out-of-core stencil loop-chain engine (arXiv 1709.02125).

Python mirror of the reference's OPS-style runtime API (proj/include/ooc/runtime.hpp,
proj/include/ooc/chain_file.hpp) over the C ABI in include/ooc_stencil.h. Every
call goes to libooc.so (C++ planner / lazy runtime / streaming engine) and
liboocdev.so (sm_100a kernels, CUDA streams); nothing computes in Python.

    rt = Runtime(executor="explicit", capacity=problem_bytes // 3)
    u = rt.declare("u", (0, 0), (n, n), halo=(1, 1), fill="(+ 1 (* 0.001 i))")
    t = rt.declare("tmp", (0, 0), (n, n), halo=(1, 1))
    rt.enqueue_loop((1, 1), (n - 1, n - 1),
                    [(u, STAR5, READ), (t, POINT, WRITE)],
                    writes={1: "(* 0.25 (+ (+ (r 0 -1 0) (r 0 1 0)) (+ (r 0 0 -1) (r 0 0 1))))"})
    values = rt.fetch_dataset(t)
"""
from __future__ import annotations

import ctypes
import json
from typing import Dict, Iterable, Optional, Sequence, Tuple

import numpy as np

from . import _native

READ, WRITE, READ_WRITE = "READ", "WRITE", "READ_WRITE"
_MODES = {READ: 0, WRITE: 1, READ_WRITE: 2}
_REDUCE = {None: 0, "SUM": 1, "MIN": 2, "MAX": 3}
EXECUTORS = {"reference": 0, "explicit": 2, "tiled_explicit": 2, "resident": 4, "plan_only": 5}
POINT = [(0, 0, 0)]


def star(ndim, radius=1):
    """Stencil::star (proj/include/ooc/stencil.hpp:28-41)."""
    offs = [(0, 0, 0)]
    for d in range(ndim):
        for o in range(-radius, radius + 1):
            if o:
                p = [0, 0, 0]
                p[d] = o
                offs.append(tuple(p))
    return offs


def line(dim, radius=1):
    """Stencil::line (proj/include/ooc/stencil.hpp:20-27)."""
    offs = []
    for o in range(-radius, radius + 1):
        p = [0, 0, 0]
        p[dim] = o
        offs.append(tuple(p))
    return offs


# ------------------------------------------------------------------ errors
class OocError(RuntimeError):
    pass


class ValidationError(OocError):
    pass


class StaleDataError(OocError):
    pass


class InfeasibleError(OocError):
    pass


class CapacityError(OocError):
    pass


class DeviceError(OocError):
    pass


_ERRORS = {-1: ValidationError, -2: StaleDataError, -3: InfeasibleError, -4: CapacityError,
           -5: DeviceError}


def _check(rc):
    if rc != 0:
        raise _ERRORS.get(rc, OocError)(_native.lib().ooc_rt_last_error().decode())


def _i64x3(v, fill):
    v = list(v) + [fill] * (3 - len(v))
    return (ctypes.c_int64 * 3)(*[int(x) for x in v])


def problem_bytes(app, nx, ny, nz=0, span=0) -> int:
    return int(_native.lib().ooc_app_problem_bytes(app.encode(), nx, ny, nz, span))


class Runtime:
    """ooc::Runtime (proj/include/ooc/runtime.hpp:53-137) on a B200."""

    def __init__(self, executor="resident", tiles=0, capacity=16_000_000_000, resident_budget=0,
                 prefetch=False, record=False, gpu=0, profile=False, arena_fill=0, tiled_dim=0,
                 fuse=True, dist=(0, 1), own=None, ghost=0, timeline=False, exact_reductions=False):
        L = _native.lib()
        o = _native.Options()
        L.ooc_rt_default_options(ctypes.byref(o))
        o.executor = EXECUTORS[executor]
        o.tiles = tiles
        o.tiled_dim = tiled_dim
        o.capacity_bytes = int(capacity)
        o.resident_budget = int(resident_budget)
        o.prefetch = int(prefetch)
        o.record_chains = int(record)
        o.gpu = gpu
        o.profile_loops = int(profile)
        o.arena_fill = arena_fill
        o.no_fuse = 0 if fuse else 1
        o.dist_rank, o.dist_world = int(dist[0]), int(dist[1])
        if own is not None:
            o.own_lo, o.own_hi = int(own[0]), int(own[1])
        o.ghost = int(ghost)
        o.timeline = int(timeline)
        h = ctypes.c_void_p()
        _check(L.ooc_rt_create(ctypes.byref(o), ctypes.byref(h)))
        self._h = h
        self.executor = executor
        if exact_reductions:
            self.set_exact_reductions(True)
        self._shapes: Dict[int, Tuple[int, int, int]] = {}

    def close(self):
        if getattr(self, "_h", None):
            _native.lib().ooc_rt_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---------------------------------------------------------------- datasets
    def declare(self, name, lo, hi, halo=(0, 0, 0), fill=0.0, elem_bytes=8) -> int:
        """Runtime::declare / declare_dataset (proj/src/dataset.cpp:5-38). `fill` is a
        number, a prefix expression over i,j,k, or an array over the allocation."""
        ndim = len(lo)
        out = ctypes.c_int()
        init = None
        expr = None
        value = 0.0
        if isinstance(fill, str):
            expr = fill.encode()
        elif isinstance(fill, np.ndarray):
            init = np.ascontiguousarray(fill, dtype=np.float64)
        else:
            value = float(fill)
        _check(_native.lib().ooc_rt_declare(
            self._h, name.encode(), ndim, _i64x3(lo, 0), _i64x3(hi, 1), _i64x3(halo, 0),
            elem_bytes, expr, value,
            init.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if init is not None else None,
            ctypes.byref(out)))
        return out.value

    def find(self, name) -> int:
        return _native.lib().ooc_rt_find_dataset(self._h, name.encode())

    @property
    def num_datasets(self) -> int:
        return _native.lib().ooc_rt_num_datasets(self._h)

    def dataset_info(self, d):
        n = ctypes.c_int64()
        stale = ctypes.c_int()
        nd = ctypes.c_int()
        lo = (ctypes.c_int64 * 3)()
        hi = (ctypes.c_int64 * 3)()
        _check(_native.lib().ooc_rt_dataset_info(self._h, d, ctypes.byref(n), ctypes.byref(stale),
                                                 ctypes.byref(nd), lo, hi))
        shape = tuple(hi[k] - lo[k] for k in range(3))
        return {"len": n.value, "stale": bool(stale.value), "ndim": nd.value,
                "lo": tuple(lo), "hi": tuple(hi), "shape": shape}

    def host(self, d) -> np.ndarray:
        """Zero-copy view of the pinned host storage (no flush, no copy-back)."""
        p = ctypes.POINTER(ctypes.c_double)()
        n = ctypes.c_int64()
        _check(_native.lib().ooc_rt_host_data(self._h, d, ctypes.byref(p), ctypes.byref(n)))
        shape = self.dataset_info(d)["shape"]
        return np.ctypeslib.as_array(p, shape=(n.value,)).reshape(shape)

    # ---------------------------------------------------------------- loops
    def enqueue_loop(self, lo, hi, args, writes=None, reduction=None):
        """Runtime::enqueue_loop (proj/src/runtime.cpp:5-11).
        args: [(dataset_id, stencil_offsets, mode)]; writes: {arg: prefix expr};
        reduction: (op in SUM/MIN/MAX, prefix expr, name)."""
        ndim = len(lo)
        nargs = len(args)
        ds = (ctypes.c_int * max(nargs, 1))(*[a[0] for a in args])
        modes = (ctypes.c_int * max(nargs, 1))(*[_MODES[a[2]] for a in args])
        nofs = (ctypes.c_int * max(nargs, 1))(*[len(a[1]) for a in args])
        flat = [int(x) for a in args for o in a[1] for x in (list(o) + [0, 0, 0])[:3]]
        offs = (ctypes.c_int64 * max(len(flat), 1))(*flat)
        writes = writes or {}
        wa = (ctypes.c_int * max(len(writes), 1))(*[int(k) for k in writes])
        we = (ctypes.c_char_p * max(len(writes), 1))(*[v.encode() for v in writes.values()])
        rop, rexpr, rname = _REDUCE[None], None, None
        if reduction:
            rop, rexpr, rname = _REDUCE[reduction[0]], reduction[1].encode(), reduction[2].encode()
        _check(_native.lib().ooc_rt_enqueue_loop(
            self._h, ndim, _i64x3(lo, 0), _i64x3(hi, 1), nargs, ds, modes, nofs, offs,
            len(writes), wa, we, rop, rexpr, rname))

    def flush(self):
        _check(_native.lib().ooc_rt_flush(self._h))

    def finish(self):
        _check(_native.lib().ooc_rt_finish(self._h))

    def sync(self):
        _check(_native.lib().ooc_rt_sync(self._h))

    def set_cyclic_flag(self, on=True):
        _check(_native.lib().ooc_rt_set_cyclic(self._h, int(bool(on))))

    def set_exact_reductions(self, on=True):
        """Debug mode: reductions folded in the reference's sequential row-major order
        (proj/src/kernel_exec.cpp:193-197), bitwise equal to it; slower (one thread per
        fold), single rank only."""
        _check(_native.lib().ooc_rt_set_exact_reductions(self._h, int(bool(on))))

    def fetch_dataset(self, d) -> np.ndarray:
        """Runtime::fetch_dataset (proj/src/runtime.cpp:13-19): flush, stale check, copy."""
        info = self.dataset_info(d)
        out = np.empty(info["shape"], dtype=np.float64)
        _check(_native.lib().ooc_rt_fetch_dataset(
            self._h, d, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), out.size))
        return out

    def fetch_reduction(self, name) -> float:
        v = ctypes.c_double()
        _check(_native.lib().ooc_rt_fetch_reduction(self._h, name.encode(), ctypes.byref(v)))
        return v.value

    # ---------------------------------------------------------------- apps
    def run_app(self, name, nx, ny, nz=0, iters=10, span=0, cyclic=False):
        """run_app (proj/src/apps.cpp:219-228) + the 3-D analogues."""
        _check(_native.lib().ooc_rt_run_app(self._h, name.encode(), nx, ny, nz, iters, span,
                                            int(cyclic)))

    def declare_app(self, name, nx, ny, nz=0, span=0):
        _check(_native.lib().ooc_rt_declare_app(self._h, name.encode(), nx, ny, nz, span))

    def app_iterations(self, name, nx, ny, nz=0, it0=0, it1=1, span=0, cyclic=False):
        """Enqueue iterations [it0, it1) of a declared app (with its own flushes)."""
        _check(_native.lib().ooc_rt_app_iterations(self._h, name.encode(), nx, ny, nz, span,
                                                   int(cyclic), it0, it1))

    # ---------------------------------------------------------------- timing
    def mark(self) -> int:
        """CUDA event on the compute queue after all work issued so far (incl. downloads)."""
        rc = _native.lib().ooc_rt_mark(self._h)
        if rc < 0:
            _check(rc)
        return rc

    def elapsed(self, a, b) -> float:
        s = ctypes.c_double()
        _check(_native.lib().ooc_rt_mark_elapsed(self._h, a, b, ctypes.byref(s)))
        return s.value

    # ---------------------------------------------------------------- introspection
    def _json(self, fn, *args):
        s = fn(self._h, *args).decode()
        v = json.loads(s)
        if isinstance(v, dict) and "error" in v:
            kind = v["error"].split(":", 1)[0]
            raise {"ValidationError": ValidationError, "InfeasibleError": InfeasibleError,
                   "CapacityError": CapacityError, "DeviceError": DeviceError,
                   "StaleDataError": StaleDataError}.get(kind, OocError)(v["error"])
        return v

    def flush_log(self):
        return self._json(_native.lib().ooc_rt_flush_log_json)

    def audit(self):
        return self._json(_native.lib().ooc_rt_audit_json)

    def report(self):
        return self._json(_native.lib().ooc_rt_report_json)

    def _csv(self, fn, *args):
        s = fn(self._h, *args)
        if s is None:
            msg = _native.lib().ooc_rt_last_error().decode()
            raise {"ValidationError": ValidationError, "InfeasibleError": InfeasibleError,
                   "CapacityError": CapacityError, "DeviceError": DeviceError,
                   "StaleDataError": StaleDataError}.get(msg.split(":", 1)[0], OocError)(msg)
        return s.decode()

    def report_csv(self, app="", size="", iters=0):
        """proj/src/metrics.cpp:46-60 schema (#oocstencil-report-v1)."""
        return self._csv(_native.lib().ooc_rt_report_csv, app.encode(), str(size).encode(), int(iters))

    def loops_csv(self):
        return self._csv(_native.lib().ooc_rt_loops_csv)

    def audit_csv(self):
        return self._csv(_native.lib().ooc_rt_audit_csv)

    def timeline_csv(self):
        """Measured command timeline (timeline=True runs), proj/src/command.cpp:160-168 schema."""
        return self._csv(_native.lib().ooc_rt_timeline_csv)

    def chain_timings(self):
        return self._json(_native.lib().ooc_rt_chain_timings_json)

    def loop_metrics(self):
        return self._json(_native.lib().ooc_rt_loop_metrics_json)

    def launch_log(self):
        """profile=True runs: [first_loop_id, n_loops, metric_bytes, seconds] per launch."""
        return self._json(_native.lib().ooc_rt_launch_log_json)

    def device(self):
        return self._json(_native.lib().ooc_rt_device_json)

    def num_chains(self):
        return _native.lib().ooc_rt_num_chains(self._h)

    def chain_plan(self, chain, tiles=0, budget=0, dump=False):
        return self._json(_native.lib().ooc_rt_chain_plan_json, chain, tiles, budget, int(dump))

    def chain_plan_text(self, chain, tiles):
        return _native.lib().ooc_rt_chain_plan_text(self._h, chain, tiles).decode()

    # ---------------------------------------------------------------- slab decomposition
    def comm_init(self, unique_id: bytes):
        """Join the NCCL communicator of the slab decomposition (128-byte id)."""
        _check(_native.lib().ooc_rt_comm_init(self._h, unique_id))

    def comm_init_ipc(self, name: str):
        """Join the CUDA-IPC transport of the slab decomposition (ranks of one node,
        same `name` on every rank; ranks may share a GPU)."""
        _check(_native.lib().ooc_rt_comm_init_ipc(self._h, name.encode()))

    def chain_export(self, chain):
        """A recorded chain's loops as this rank runs them (window-clipped)."""
        return self._json(_native.lib().ooc_rt_chain_export_json, chain)

    def dist_plan(self, chain):
        """Ghost depth the chain needs and the ghost-band exchange it triggers."""
        return self._json(_native.lib().ooc_rt_dist_plan_json, chain)

    def chain_jit_check(self, chain, fuse=True):
        """Compile (NVRTC, sm_100a, no GPU needed) the specialised kernels of a recorded chain."""
        return self._json(_native.lib().ooc_rt_chain_jit_check, chain, int(fuse))

    def chain_sweep_check(self, chain, compile=True):
        """Row-sweep runs of a recorded chain with their plans (lags, halos, rings);
        compile=True builds each run's kernel for sm_100a (NVRTC, no GPU needed)."""
        out = self._json(_native.lib().ooc_rt_chain_sweep_check, chain, int(compile))
        for g in out:
            if g["ok"] and g["plan"].startswith("{"):
                g["plan"] = json.loads(g["plan"].split("\n")[0])
        return out

    def chain_oracle(self, chain, tiles):
        return self._json(_native.lib().ooc_rt_chain_oracle_json, chain, tiles)


# ---------------------------------------------------------------------- chain files
def load_program(rt: Runtime, prog):
    """Chain-file loader (proj/src/chain_file.cpp:58-162, load_chain_json): declare the
    datasets, then enqueue the loops; an optional "ops" list interleaves flush / cyclic /
    finish. Parsed and executed natively (csrc/host/chain_file.cpp)."""
    text = prog if isinstance(prog, str) else json.dumps(prog)
    n = ctypes.c_int()
    _check(_native.lib().ooc_rt_load_chain_json(rt._h, text.encode(), ctypes.byref(n)))
    return rt


__all__ = ["Runtime", "load_program", "problem_bytes", "star", "line", "POINT", "READ", "WRITE",
           "READ_WRITE", "ValidationError", "StaleDataError", "InfeasibleError", "CapacityError",
           "DeviceError", "OocError"]


def set_jit(mode: int, min_points: int = -1) -> None:
    """Specialised-kernel policy (include/ooc_device.h ooc_jit_config): 0 interpreter
    only, 1 specialise launches of >= min_points points, 2 always specialise."""
    _native.lib()
    dev = ctypes.CDLL(_native.device_lib_path())
    dev.ooc_jit_config.argtypes = [ctypes.c_int, ctypes.c_longlong]
    rc = dev.ooc_jit_config(mode, min_points)
    if rc != 0:
        raise OocError("ooc_jit_config failed")


def set_sweep(on: bool) -> None:
    """Process-wide: row-sweep kernels for resident untiled 2-D chains (ooc_rt_set_sweep)."""
    _native.lib().ooc_rt_set_sweep(int(bool(on)))


def set_sweep_3d(on: bool) -> None:
    """Process-wide: 3-D chains as plane-tile row sweeps (ooc_sweep_set_3d)."""
    _native.lib()
    dev = ctypes.CDLL(_native.device_lib_path())
    dev.ooc_sweep_set_3d(int(bool(on)))


def set_row_recompute(on: bool) -> None:
    """Process-wide fusion policy (ooc_rt_set_row_recompute)."""
    _native.lib().ooc_rt_set_row_recompute(int(bool(on)))


def jit_report():
    """Autotuned tile shape of every specialised kernel (ooc_jit_report)."""
    _native.lib()
    dev = ctypes.CDLL(_native.device_lib_path())
    buf = ctypes.create_string_buffer(1 << 16)
    dev.ooc_jit_report(buf, 1 << 16)
    return json.loads(buf.value.decode())


def sweep_report():
    """Prefetch depth autotuned per row-sweep structure (ooc_sweep_report)."""
    _native.lib()
    dev = ctypes.CDLL(_native.device_lib_path())
    buf = ctypes.create_string_buffer(1 << 16)
    dev.ooc_sweep_report(buf, 1 << 16)
    return json.loads(buf.value.decode())


def jit_status() -> str:
    _native.lib()
    dev = ctypes.CDLL(_native.device_lib_path())
    buf = ctypes.create_string_buffer(256)
    dev.ooc_jit_status(buf, 256)
    return buf.value.decode()
