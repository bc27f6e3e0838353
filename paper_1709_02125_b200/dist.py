"""Slab decomposition across GPUs (north_star (e)): one process and one Runtime per
GPU, dimension 0 split into contiguous owned slabs, `ghost` rows recomputed on each
side, ghost bands refreshed by NCCL point-to-point after every chain and reductions
all-reduced — all inside the runtime (csrc/host/runtime.cpp, csrc/device/comm.cu).
torch.distributed is only the bootstrap that carries NCCL's unique id.
"""
from __future__ import annotations

import ctypes
import os
import uuid

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


def transport() -> str:
    """Ghost-exchange transport of the slab decomposition: "nccl" (default) or "ipc"
    (CUDA IPC peer copies + a shared-memory rendezvous; OOC_COMM=ipc)."""
    t = os.environ.get("OOC_COMM", "nccl").lower()
    if t not in ("nccl", "ipc"):
        raise ValueError(f"OOC_COMM={t}: expected nccl or ipc")
    return t


def ipc_name() -> str:
    """A job-unique rendezvous name for the IPC transport."""
    return f"{os.getpid()}_{uuid.uuid4().hex[:12]}"


def init_comm(rt: Runtime, rank: int, group=None, kind: str | None = None):
    """Join the slab decomposition's communicator. NCCL: rank 0 creates the id and
    torch.distributed broadcasts it. IPC: rank 0 picks the rendezvous name and
    torch.distributed broadcasts that. torch is only the bootstrap either way."""
    import torch.distributed as dist
    kind = kind or transport()
    if kind == "ipc":
        obj = [ipc_name() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        rt.comm_init_ipc(obj[0])
        return
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
