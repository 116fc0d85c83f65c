"""Seeded synthetic inputs for the sparse embedding layer (shared by oracle tests and the GPU path).

This module holds NO arithmetic of the method (no keys, dedup, routing, pooling or optimizer math):
it only draws ids, CSR offsets and upstream gradients dY with the shapes and distributions of the
workloads named in BASELINE.json `configs` (BJ:7-11), following the recipe of SURVEY.md §8(d) and
the readings R17-R20 listed in DESIGN.md §3.

Recipe:
  * seeds: numpy SeedSequence([2112, cfg_index, rank, step]) for ids/offsets, [..., 1] for dY;
  * Zipf(s) ids: rank k ~ Generator.zipf(s) truncated to 1..R by rejection, then
    id = ((k - 1) * 2654435761 + c_t) mod R  (a bijection since 2654435761 is prime, gcd(A, R) = 1),
    so hot ids scatter across shards; c_t = (t * 40503 + 17) mod R;
  * uniform ids: integers in [0, R);
  * hot-id stress (C5, R20): per table, 90% uniform over the table's top-1000 permuted ranks, 10% uniform
    over the rest;
  * bag lengths: C1 U{1..8}; C2-C4 exactly 1 (one categorical value per Criteo field, R18); C5 exactly 64;
  * dY ~ U[-1, 1) float32.
CSR layout: slot-major, bag (s, b) = ids[offsets[s*B+b] : offsets[s*B+b+1]].
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import List, Optional

import numpy as np

PERM_A = 2654435761  # prime; coprime to every table size used below


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config (per GPU / per rank quantities)."""
    name: str
    index: int                      # cfg index used in the seed
    rows: tuple                     # rows per table
    dim: int
    slot_table: tuple               # slot -> table
    batch: int                      # per-rank batch (R17)
    bag: str                        # "u1_8" | "fixed"
    bag_len: int                    # for "fixed"
    ids: str                        # "uniform" | "zipf" | "hot1k"
    zipf_s: float = 1.05
    pool: str = "sum"               # "sum" | "mean"
    opt: str = "adagrad"            # "sgd" | "adagrad" | "rowwise_adagrad"
    lr: float = 0.01
    eps: float = 1e-6               # R13
    init_accum: float = 0.0         # R13
    world: int = 1
    seed: int = 2112

    @property
    def num_slots(self) -> int:
        return len(self.slot_table)

    @property
    def num_tables(self) -> int:
        return len(self.rows)

    @property
    def total_rows(self) -> int:
        return int(sum(self.rows))

    def with_(self, **kw) -> "Workload":
        return replace(self, **kw)


def _c3_rows():
    # 100M rows split over 26 tables: 3,846,154 each except the last absorbs the remainder
    r = [3_846_154] * 26
    r[-1] = 100_000_000 - 3_846_154 * 25
    return tuple(r)


WORKLOADS = {
    # BJ:7  "1 table 100k rows x dim 16, 4 slots, batch 1024, bag<=8, uniform ids, SGD, 1 GPU"
    "C1": Workload("C1", 1, (100_000,), 16, (0, 0, 0, 0), 1024, "u1_8", 0, "uniform", opt="sgd"),
    # BJ:8  "Criteo-like: 26 slots, 10M rows/table, dim 64, batch 16k, Zipf(1.05) ids, Adagrad, 1 GPU"
    "C2": Workload("C2", 2, (10_000_000,) * 26, 64, tuple(range(26)), 16384, "fixed", 1, "zipf", 1.05),
    # BJ:9  "Criteo-like 26 slots, 100M total rows, dim 64, row-sharded over 2/4/8 GPUs with all-to-all"
    "C3": Workload("C3", 3, _c3_rows(), 64, tuple(range(26)), 16384, "fixed", 1, "zipf", 1.05),
    # BJ:10 "large table 1B rows x dim 128 fp32 sharded over 8xB200, batch 64k, Zipf(1.2), Adagrad" (R19: 26 slots -> 1 table)
    "C4": Workload("C4", 4, (1_000_000_000,), 128, (0,) * 26, 65536, "fixed", 1, "zipf", 1.2, world=8),
    # C4-half (BJ:10 at the 4 GPUs gpurun offers): the same structure on 5e8 rows
    "C4h": Workload("C4h", 4, (500_000_000,), 128, (0,) * 26, 65536, "fixed", 1, "zipf", 1.2, world=4),
    # BJ:11 "hot-id stress: 26 slots, bag 64, 90% of ids from top-1k rows, 8 GPUs" (R20)
    "C5": Workload("C5", 5, _c3_rows(), 64, tuple(range(26)), 16384, "fixed", 64, "hot1k", world=8),
}


@dataclass
class Batch:
    """One rank's CSR batch: ids int64 [nnz], offsets int64 [S*B+1] (slot-major), dY float32 [B][S][D] or None."""
    ids: np.ndarray
    offsets: np.ndarray
    batch: int
    dy: Optional[np.ndarray] = None

    @property
    def nnz(self) -> int:
        return int(self.offsets[-1])


def _rng(wl: Workload, rank: int, step: int, stream: int = 0) -> np.random.Generator:
    key = [2112, wl.index, rank, step] + ([stream] if stream else [])
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(key)))


def bag_lengths(wl: Workload, rng: np.random.Generator, batch: int) -> np.ndarray:
    n = wl.num_slots * batch
    if wl.bag == "u1_8":
        return rng.integers(1, 9, size=n, dtype=np.int64)
    return np.full(n, wl.bag_len, dtype=np.int64)


def _zipf_ranks(rng: np.random.Generator, s: float, R: int, n: int) -> np.ndarray:
    """k ~ Zipf(s) conditioned on k <= R (rejection; exactly the truncated law)."""
    out = np.empty(n, dtype=np.int64)
    filled = 0
    while filled < n:
        need = n - filled
        k = rng.zipf(s, size=int(need * 1.8) + 64)
        k = k[(k >= 1) & (k <= R)]
        take = min(need, k.size)
        out[filled:filled + take] = k[:take]
        filled += take
    return out


def permute_rank(k: np.ndarray, R: int, t: int) -> np.ndarray:
    """Scatter Zipf rank k (1-based) over [0, R): ((k-1)*A + c_t) mod R."""
    c_t = (t * 40503 + 17) % R
    k = k.astype(np.uint64)
    return ((((k - np.uint64(1)) % np.uint64(R)) * np.uint64(PERM_A % R) + np.uint64(c_t)) % np.uint64(R)).astype(np.int64)


def draw_ids(wl: Workload, rng: np.random.Generator, t: int, n: int) -> np.ndarray:
    R = wl.rows[t]
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    if wl.ids == "uniform":
        return rng.integers(0, R, size=n, dtype=np.int64)
    if wl.ids == "zipf":
        return permute_rank(_zipf_ranks(rng, wl.zipf_s, R, n), R, t)
    if wl.ids == "hot1k":
        hot = min(1000, R)
        is_hot = rng.random(n) < 0.9
        k = np.where(is_hot,
                     rng.integers(1, hot + 1, size=n),
                     rng.integers(hot + 1, max(hot + 2, R + 1), size=n) if R > hot else rng.integers(1, hot + 1, size=n))
        return permute_rank(k, R, t)
    raise ValueError(wl.ids)


def make_batch(wl: Workload, rank: int = 0, step: int = 0, batch: Optional[int] = None,
               with_dy: bool = True, empty_frac: float = 0.0) -> Batch:
    """Generate one rank's batch. `batch` overrides wl.batch (reduced parity sizes); `empty_frac`
    zeroes that fraction of bag lengths (edge-case tests)."""
    B = wl.batch if batch is None else int(batch)
    rng = _rng(wl, rank, step)
    lens = bag_lengths(wl, rng, B)
    if empty_frac > 0:
        lens[rng.random(lens.size) < empty_frac] = 0
    offsets = np.zeros(lens.size + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    ids = np.empty(int(offsets[-1]), dtype=np.int64)
    for s in range(wl.num_slots):
        lo, hi = offsets[s * B], offsets[(s + 1) * B]
        ids[lo:hi] = draw_ids(wl, rng, wl.slot_table[s], int(hi - lo))
    dy = None
    if with_dy:
        dy = make_dy(wl, rank, step, B)
    return Batch(ids=ids, offsets=offsets, batch=B, dy=dy)


def make_dy(wl: Workload, rank: int, step: int, batch: int) -> np.ndarray:
    rng = _rng(wl, rank, step, stream=1)
    return (rng.random((batch, wl.num_slots, wl.dim), dtype=np.float32) * 2.0 - 1.0).astype(np.float32)
