"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes binding of oracle/_ref/libooc_ref.so: the unmodified reference library
(/root/reference/proj/src, compiled by oracle/ref/Makefile) behind the small C
wrapper oracle/ref/ref_capi.cpp. Used to generate golden vectors, to pin the
numpy restatement (oracle/ooc_oracle.py), and as bench.py's CPU baseline
("kind": "reference"). Never imported by the product package.
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libooc_ref.so")

EXECUTORS = {"reference": 0, "cache": 1, "explicit": 2, "unified": 3}

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle/ref`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i, ll, cp, dp = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_char_p, \
            ctypes.POINTER(ctypes.c_double)
        sig = {
            "refo_last_error": (cp, []),
            "refo_create": (vp, [i, i, ll, i, i, i]),
            "refo_destroy": (None, [vp]),
            "refo_load_program": (i, [vp, cp]),
            "refo_run_app": (i, [vp, cp, ll, ll, i, i, i]),
            "refo_app_problem_bytes": (ll, [cp, ll, ll, i]),
            "refo_flush": (i, [vp]),
            "refo_finish": (i, [vp]),
            "refo_num_datasets": (i, [vp]),
            "refo_dataset_name": (cp, [vp, i]),
            "refo_dataset_len": (ll, [vp, i]),
            "refo_dataset_stale": (i, [vp, i]),
            "refo_copy_dataset": (i, [vp, i, dp]),
            "refo_dataset_ptr": (dp, [vp, i]),
            "refo_fetch_dataset": (i, [vp, i, dp]),
            "refo_fetch_reduction": (i, [vp, cp, dp]),
            "refo_totals": (i, [vp, ctypes.POINTER(ll), dp]),
            "refo_flush_log_json": (cp, [vp]),
            "refo_audit_json": (cp, [vp]),
            "refo_num_chains": (i, [vp]),
            "refo_chain_plan_json": (cp, [vp, i, i, ll]),
            "refo_chain_plan_dump_json": (cp, [vp, i, i]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code
        self.kind = msg.split(":", 1)[0]


class RefRuntime:
    """Reference ooc::Runtime (proj/include/ooc/runtime.hpp:53-137)."""

    def __init__(self, executor="reference", tiles=0, capacity=0, openmp=True, prefetch=False,
                 record=False):
        L = lib()
        self._h = L.refo_create(EXECUTORS[executor], tiles, capacity, int(openmp), int(prefetch),
                                int(record))

    def close(self):
        if self._h:
            lib().refo_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            raise RefError(rc, lib().refo_last_error().decode())

    def load_program(self, prog):
        text = prog if isinstance(prog, str) else json.dumps(prog)
        self._check(lib().refo_load_program(self._h, text.encode()))
        return self

    def run_app(self, name, nx, ny, iters, span=0, cyclic=False):
        self._check(lib().refo_run_app(self._h, name.encode(), nx, ny, iters, span, int(cyclic)))
        return self

    def flush(self):
        self._check(lib().refo_flush(self._h))

    def finish(self):
        self._check(lib().refo_finish(self._h))

    def datasets(self):
        n = lib().refo_num_datasets(self._h)
        return [lib().refo_dataset_name(self._h, d).decode() for d in range(n)]

    def host(self, d) -> np.ndarray:
        n = lib().refo_dataset_len(self._h, d)
        out = np.empty(n, dtype=np.float64)
        lib().refo_copy_dataset(self._h, d, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        return out

    def host_view(self, d) -> np.ndarray:
        """Zero-copy view of the reference's host buffer (valid until close())."""
        n = lib().refo_dataset_len(self._h, d)
        return np.ctypeslib.as_array(lib().refo_dataset_ptr(self._h, d), shape=(n,))

    def stale(self, d) -> bool:
        return bool(lib().refo_dataset_stale(self._h, d))

    def fetch_dataset(self, d) -> np.ndarray:
        n = lib().refo_dataset_len(self._h, d)
        out = np.empty(n, dtype=np.float64)
        self._check(lib().refo_fetch_dataset(self._h, d,
                                             out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def fetch_reduction(self, name) -> float:
        v = ctypes.c_double()
        self._check(lib().refo_fetch_reduction(self._h, name.encode(), ctypes.byref(v)))
        return v.value

    def totals(self):
        arr = (ctypes.c_longlong * 8)()
        t = ctypes.c_double()
        lib().refo_totals(self._h, arr, ctypes.byref(t))
        return {"uploaded": arr[0], "downloaded": arr[1], "d2d": arr[2], "metric_bytes": arr[3],
                "chains": arr[4], "last_tiles": arr[5], "loop_time_s": t.value}

    def flush_log(self):
        return json.loads(lib().refo_flush_log_json(self._h).decode())

    def audit(self):
        return json.loads(lib().refo_audit_json(self._h).decode())

    def num_chains(self):
        return lib().refo_num_chains(self._h)

    def chain_plan(self, chain_index, tiles=0, budget=0):
        return json.loads(lib().refo_chain_plan_json(self._h, chain_index, tiles, budget).decode())

    def chain_plan_dump(self, chain_index, tiles):
        return json.loads(lib().refo_chain_plan_dump_json(self._h, chain_index, tiles).decode())


def app_problem_bytes(name, nx, ny, span=0) -> int:
    return lib().refo_app_problem_bytes(name.encode(), nx, ny, span)
