"""ctypes binding of libooc.so (the C ABI in include/ooc_stencil.h).

The native library is mandatory: importing this module without it raises, and
there is no Python/CPU execution path behind it.
"""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(PKG, "lib")
LIB_PATH = os.path.join(LIB_DIR, "libooc.so")


class NativeLibraryMissing(ImportError):
    pass


class Options(ctypes.Structure):
    _fields_ = [
        ("executor", ctypes.c_int),
        ("tiles", ctypes.c_int),
        ("tiled_dim", ctypes.c_int),
        ("capacity_bytes", ctypes.c_longlong),
        ("resident_budget", ctypes.c_longlong),
        ("prefetch", ctypes.c_int),
        ("record_chains", ctypes.c_int),
        ("gpu", ctypes.c_int),
        ("profile_loops", ctypes.c_int),
        ("arena_fill", ctypes.c_int),
        ("no_fuse", ctypes.c_int),
        ("dist_rank", ctypes.c_int),
        ("dist_world", ctypes.c_int),
        ("own_lo", ctypes.c_longlong),
        ("own_hi", ctypes.c_longlong),
        ("ghost", ctypes.c_longlong),
        ("timeline", ctypes.c_int),
    ]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} is missing: build it with `python -m paper_1709_02125_b200.build` "
            "(or __graft_entry__.build()); ooc-b200 has no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)  # RTLD_LOCAL: keep the ooc:: C++ symbols private
    vp, i, i64, cp, dp = (ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_char_p,
                          ctypes.POINTER(ctypes.c_double))
    I64P = ctypes.POINTER(ctypes.c_int64)
    IP = ctypes.POINTER(ctypes.c_int)
    sig = {
        "ooc_rt_default_options": (None, [ctypes.POINTER(Options)]),
        "ooc_rt_last_error": (cp, []),
        "ooc_rt_create": (i, [ctypes.POINTER(Options), ctypes.POINTER(vp)]),
        "ooc_rt_destroy": (None, [vp]),
        "ooc_rt_declare": (i, [vp, cp, i, I64P, I64P, I64P, i64, cp, ctypes.c_double, dp, IP]),
        "ooc_rt_enqueue_loop": (i, [vp, i, I64P, I64P, i, IP, IP, IP, I64P, i, IP,
                                    ctypes.POINTER(cp), i, cp, cp]),
        "ooc_rt_flush": (i, [vp]),
        "ooc_rt_finish": (i, [vp]),
        "ooc_rt_sync": (i, [vp]),
        "ooc_rt_set_cyclic": (i, [vp, i]),
        "ooc_rt_set_exact_reductions": (i, [vp, i]),
        "ooc_rt_fetch_dataset": (i, [vp, i, dp, i64]),
        "ooc_rt_fetch_reduction": (i, [vp, cp, dp]),
        "ooc_rt_num_datasets": (i, [vp]),
        "ooc_rt_dataset_info": (i, [vp, i, I64P, IP, IP, I64P, I64P]),
        "ooc_rt_find_dataset": (i, [vp, cp]),
        "ooc_rt_host_data": (i, [vp, i, ctypes.POINTER(dp), I64P]),
        "ooc_rt_run_app": (i, [vp, cp, i64, i64, i64, i, i, i]),
        "ooc_rt_declare_app": (i, [vp, cp, i64, i64, i64, i]),
        "ooc_app_problem_bytes": (i64, [cp, i64, i64, i64, i]),
        "ooc_rt_app_iterations": (i, [vp, cp, i64, i64, i64, i, i, i, i]),
        "ooc_rt_mark": (i, [vp]),
        "ooc_rt_mark_elapsed": (i, [vp, i, i, dp]),
        "ooc_rt_flush_log_json": (cp, [vp]),
        "ooc_rt_audit_json": (cp, [vp]),
        "ooc_rt_report_json": (cp, [vp]),
        "ooc_rt_report_csv": (cp, [vp, cp, cp, ctypes.c_int]),
        "ooc_rt_loops_csv": (cp, [vp]),
        "ooc_rt_set_row_recompute": (None, [i]),
        "ooc_rt_set_sweep": (None, [i]),
        "ooc_rt_audit_csv": (cp, [vp]),
        "ooc_rt_timeline_csv": (cp, [vp]),
        "ooc_rt_chain_timings_json": (cp, [vp]),
        "ooc_rt_loop_metrics_json": (cp, [vp]),
        "ooc_rt_device_json": (cp, [vp]),
        "ooc_rt_launch_log_json": (cp, [vp]),
        "ooc_rt_num_chains": (i, [vp]),
        "ooc_rt_chain_plan_json": (cp, [vp, i, i, i64, i]),
        "ooc_rt_chain_plan_text": (cp, [vp, i, i]),
        "ooc_rt_chain_jit_check": (cp, [vp, i, i]),
        "ooc_rt_chain_sweep_check": (cp, [vp, i, i]),
        "ooc_rt_comm_init": (i, [vp, ctypes.c_char_p]),
        "ooc_rt_comm_init_ipc": (i, [vp, ctypes.c_char_p]),
        "ooc_rt_load_chain_json": (i, [vp, ctypes.c_char_p, ctypes.POINTER(i)]),
        "ooc_rt_chain_export_json": (cp, [vp, i]),
        "ooc_rt_dist_plan_json": (cp, [vp, i]),
        "ooc_rt_chain_oracle_json": (cp, [vp, i, i]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def device_lib_path():
    return os.path.join(LIB_DIR, "liboocdev.so")
