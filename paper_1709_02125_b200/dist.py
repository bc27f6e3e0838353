"""Slab decomposition across GPUs (north_star (e)): one process and one Runtime per
GPU, dimension 0 split into contiguous owned slabs, `ghost` rows recomputed on each
side, ghost bands refreshed by NCCL point-to-point after every chain and reductions
all-reduced — all inside the runtime (csrc/host/runtime.cpp, csrc/device/comm.cu).
torch.distributed is only the bootstrap that carries NCCL's unique id.
"""
from __future__ import annotations

import ctypes

from . import Runtime, _native


def slab(rank: int, world: int, rows: int, origin: int = 0):
    """Owned rows [lo, hi) of `rank` for `rows` rows starting at `origin` (balanced)."""
    lo = origin + (rows * rank) // world
    hi = origin + (rows * (rank + 1)) // world
    return lo, hi


def unique_id() -> bytes:
    _native.lib()
    dev = ctypes.CDLL(_native.device_lib_path())
    buf = ctypes.create_string_buffer(128)
    rc = dev.ooc_comm_unique_id(buf)
    if rc != 0:
        dev.ooc_dev_last_error.restype = ctypes.c_char_p
        raise RuntimeError("ooc_comm_unique_id: " + dev.ooc_dev_last_error().decode())
    return buf.raw


def init_comm(rt: Runtime, rank: int, group=None):
    """Rank 0 creates the NCCL id, torch.distributed broadcasts it, every rank joins."""
    import torch.distributed as dist
    obj = [unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    rt.comm_init(obj[0])


def chain_depth(app: str, iters: int, span: int = 0, ndim: int = 2) -> int:
    """Ghost rows an app's chains need (the largest dependency depth of any chain);
    depends on the chain structure only, so it is computed on a small instance."""
    import paper_1709_02125_b200 as B
    n = 48 if ndim == 2 else 16
    rt = B.Runtime("plan_only", record=True, tiles=1)
    rt.run_app(app, n, n, n if ndim == 3 else 0, iters, span)
    return max(rt.dist_plan(c)["depth"] for c in range(rt.num_chains()))
