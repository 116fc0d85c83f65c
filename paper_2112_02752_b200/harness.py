"""Glue between the seeded synthetic workloads (synthgen) and the C-ABI binding: build a layer for a
BASELINE.json config and stage a batch in device memory with torch. No arithmetic of the method."""
from __future__ import annotations

from typing import Optional

import numpy as np

from .emb import EmbeddingLayer


def make_layer(wl, *, max_batch: int, max_ids: int, world: int = 1, rank: int = 0, nccl_id: Optional[bytes] = None,
               device: int = 0, shard: str = "cyclic") -> EmbeddingLayer:
    return EmbeddingLayer(wl.rows, wl.dim, wl.slot_table, pool=wl.pool, opt=wl.opt, eps=wl.eps,
                          init_accum=wl.init_accum, seed=wl.seed, max_batch=max_batch, max_ids=max_ids,
                          rank=rank, world=world, nccl_id=nccl_id, device=device, shard=shard)


class DeviceBatch:
    """A synthgen.Batch copied to device tensors (ids int64, offsets int64, dY fp32, out fp32)."""

    def __init__(self, bt, num_slots: int, dim: int, device: int = 0, pin: bool = False):
        import torch
        dev = torch.device("cuda", device)
        self.batch, self.nnz = bt.batch, bt.nnz
        self.ids = torch.from_numpy(np.ascontiguousarray(bt.ids)).to(dev)
        self.offsets = torch.from_numpy(np.ascontiguousarray(bt.offsets)).to(dev)
        self.dy = torch.from_numpy(np.ascontiguousarray(bt.dy)).to(dev) if bt.dy is not None else None
        self.out = torch.empty((bt.batch, num_slots, dim), dtype=torch.float32, device=dev)


def make_group(wl, *, world: int, max_batch: int, max_ids, devices=None, shard: str = "cyclic"):
    """All `world` ranks of a row-sharded layer in this process (emb_create_group)."""
    from .emb import EmbeddingGroup
    return EmbeddingGroup(wl.rows, wl.dim, wl.slot_table, world=world, devices=devices, pool=wl.pool, opt=wl.opt,
                          eps=wl.eps, init_accum=wl.init_accum, seed=wl.seed, max_batch=max_batch, max_ids=max_ids,
                          shard=shard)
