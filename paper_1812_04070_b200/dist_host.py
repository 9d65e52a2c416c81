"""Host-side plumbing of the multi-GPU layer (one process per GPU).

torch.distributed is used only for the bootstrap and for host-side reductions
of timings/counters (gloo or nccl process group, whichever the caller made);
the data-path exchanges run inside libsimdx.so on its own NCCL communicator.
"""
from __future__ import annotations

import os
from typing import Callable, Optional

import torch
import torch.distributed as dist


def env_rank():
    """(world, rank, local_rank) from the torchrun environment (1, 0, 0 when absent)."""
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def init_group(backend: str = "gloo") -> None:
    if dist.is_available() and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)


def broadcast_bytes(data: Optional[bytes], src: int = 0) -> bytes:
    """Rank `src` provides `data` (e.g. the 128-byte NCCL unique id); every rank returns it."""
    obj = [data]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def nccl_id_for_job(make_id: Callable[[], bytes]) -> bytes:
    """Rank 0 creates the NCCL unique id with `make_id`, everyone receives it."""
    rank = dist.get_rank()
    return broadcast_bytes(make_id() if rank == 0 else None, src=0)


def allreduce(x: float, op: str = "max") -> float:
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN}[op])
    return float(t.item())


def partition(n: int, nranks: int, rank: int):
    """Owned vertex range of `rank`: the rule of sx_dist_create (V = ceil(n/P) rounded up to 32)."""
    V = ((n + nranks - 1) // nranks + 31) // 32 * 32 or 32
    lo = min(n, rank * V)
    return lo, min(n, lo + V)


def weak_scale(base_scale: int, world: int) -> int:
    """Per-GPU work fixed: R-MAT scale base + log2(world) (2^base vertices per GPU)."""
    s = base_scale
    w = world
    while w > 1:
        assert w % 2 == 0, "weak scaling needs a power-of-two GPU count"
        s += 1
        w //= 2
    return s
