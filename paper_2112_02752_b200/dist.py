"""torch.distributed plumbing for the row-sharded (world > 1) mode: rank discovery from the torchrun
environment, the 128-byte ncclUniqueId broadcast that emb_create needs, and max-over-ranks timing.
Plumbing only: all exchanges of the embedding step run inside libemb (peer-memory kernels; NCCL only
bootstraps the CUDA IPC handles at create, or carries the v1 exchange when EMB_EXCHANGE=nccl)."""
from __future__ import annotations

import os
from typing import Callable, Optional, Tuple


def env_rank() -> Tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def share_unique_id(make_id: Callable[[], bytes], group=None) -> bytes:
    """Rank 0 creates the id (emb_get_unique_id), every rank receives the same 128 bytes."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def max_over_ranks(value: float, device: Optional[str] = None) -> float:
    """Maximum of a per-rank scalar (e.g. the device-timed region of each rank)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
