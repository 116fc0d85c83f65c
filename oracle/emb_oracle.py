"""Plain CPU oracle for the sparse distributed embedding layer — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference` legs may
import or execute anything under `oracle/`. The product path (paper_2112_02752_b200) never does; it
shares no code, header, table or constant generator with this file (the only shared module is the
seeded input generator `synthgen`, which holds none of the method's arithmetic).

What is computed (paper: the "large sparse distributed embedding lookup layer" that converts "massive
high-dimensional sparse data into dense features", §1 and PAPER.md:525-527 §3.3; the
paper gives no algorithm, so the semantics are BASELINE.json north_star (BJ:5) plus the readings
R1-R22 of SURVEY.md §8(c), restated in DESIGN.md §3):

  1. keys      g = base[t] + id,  t = slot_table[s],  base[t] = sum_{t' < t} rows[t']       (R5)
  2. forward   Y[b, s, :] = fp32( sum_{id in bag(s,b)} W_t[id, :] )  (fp64 sum; mean divides by |bag|;
               empty bag -> 0)                                                            (R1-R3)
  3. dedup     U = sorted unique {g}, counts, inverse                                      (R5, R6)
  4. routing   owner(g) = g mod W, local(g) = g div W (cyclic); block: rows_per = ceil(R/W) (R7)
  5. owner set U_o(d) = union of the send lists r -> d; owner counts = sum of rank counts
  6. backward  c_j = dY[b, s, :] (sum) or dY[b, s, :] / |bag| (mean);  G[g] = sum_j c_j in fp64 over all
               ranks (no 1/B, no 1/W)                                                     (R8-R11)
  7. update    SGD: w <- w - lr*G ;  Adagrad (element-wise, eps outside sqrt): a <- a + G^2,
               w <- w - lr*G/(sqrt(a)+eps); row-wise Adagrad (one accumulator per row, SURVEY
               §8(f) f1): a_r <- a_r + mean_c(G[c]^2), w <- w - lr*G/(sqrt(a_r)+eps); computed in
               fp64 from the fp32 state, rounded once; untouched rows bitwise unchanged   (R12-R14')
  8. init      w[g, c] = int16(splitmix64(seed XOR (g*D + c)) >> 48) * 2^-19,  a = init_accum  (R15)

Everything is the plain definition written out with NumPy primitives (np.unique, np.add.at,
fancy indexing); no blocking, fusion or reordering. Pins: tests/test_oracle_pins.py.
Parity status of every function: pinned; none is "parity unpinned".
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Sequence, Tuple

import numpy as np

MASK64 = (1 << 64) - 1
SPLITMIX_GAMMA = np.uint64(0x9E3779B97F4A7C15)
SPLITMIX_M1 = np.uint64(0xBF58476D1CE4E5B9)
SPLITMIX_M2 = np.uint64(0x94D049BB133111EB)


# ----------------------------------------------------------------------------- init (R15)
def splitmix64_next(state: np.ndarray) -> np.ndarray:
    """First output of SplitMix64 (Steele, Lea & Flood 2014) seeded with `state` (uint64 array):
    z = state + 0x9E3779B97F4A7C15; z = (z ^ z>>30)*0xBF58476D1CE4E5B9; z = (z ^ z>>27)*0x94D049BB133111EB;
    return z ^ z>>31.  (uint64 wrap-around arithmetic.)"""
    with np.errstate(over="ignore"):
        z = np.asarray(state, dtype=np.uint64) + SPLITMIX_GAMMA
        z = (z ^ (z >> np.uint64(30))) * SPLITMIX_M1
        z = (z ^ (z >> np.uint64(27))) * SPLITMIX_M2
        return z ^ (z >> np.uint64(31))


def init_weights(seed: int, g: np.ndarray, dim: int) -> np.ndarray:
    """R15: w[g, c] = int16(h >> 48) * 2^-19 with h = splitmix64(seed XOR (g*D + c)); float32 [n, D]."""
    g = np.asarray(g, dtype=np.uint64).reshape(-1)
    with np.errstate(over="ignore"):
        x = np.uint64(seed) ^ (g[:, None] * np.uint64(dim) + np.arange(dim, dtype=np.uint64)[None, :])
    h = splitmix64_next(x)
    top = (h >> np.uint64(48)).astype(np.uint16).view(np.int16).astype(np.float64)
    return (top * 2.0 ** -19).astype(np.float32)


# ----------------------------------------------------------------------------- config
@dataclass(frozen=True)
class OracleConfig:
    rows: Tuple[int, ...]          # rows per table
    dim: int
    slot_table: Tuple[int, ...]    # slot -> table
    pool: str = "sum"              # "sum" | "mean"
    opt: str = "adagrad"           # "sgd" | "adagrad" | "rowwise_adagrad"
    eps: float = 1e-6
    init_accum: float = 0.0
    seed: int = 2112
    world: int = 1
    shard: str = "cyclic"          # "cyclic" | "block"

    @property
    def base(self) -> np.ndarray:
        """base[t] = sum_{t' < t} rows[t'] (fused row space, R5)."""
        b = np.zeros(len(self.rows), dtype=np.int64)
        for t in range(1, len(self.rows)):
            b[t] = b[t - 1] + self.rows[t - 1]
        return b

    @property
    def total_rows(self) -> int:
        return int(sum(self.rows))

    @property
    def accum_width(self) -> int:
        """Optimizer state floats per row: D (element-wise Adagrad, and the unused SGD slot) or 1
        (row-wise Adagrad, R14')."""
        return 1 if self.opt == "rowwise_adagrad" else self.dim


def config_from_workload(wl, world: int = 1, shard: str = "cyclic") -> OracleConfig:
    return OracleConfig(rows=tuple(wl.rows), dim=wl.dim, slot_table=tuple(wl.slot_table), pool=wl.pool,
                        opt=wl.opt, eps=wl.eps, init_accum=wl.init_accum, seed=wl.seed, world=world, shard=shard)


# ----------------------------------------------------------------------------- step 1: keys
def occurrence_keys(cfg: OracleConfig, ids: np.ndarray, offsets: np.ndarray, batch: int):
    """For every occurrence j: its bag index s*B+b, the slot s and the fused key g = base[t(s)] + id.
    Validates the CSR (offsets[0] = 0, non-decreasing, offsets[-1] = len(ids)) and ids (R4): raises."""
    S = len(cfg.slot_table)
    ids = np.asarray(ids, dtype=np.int64)
    offsets = np.asarray(offsets, dtype=np.int64)
    if offsets.shape != (S * batch + 1,):
        raise ValueError("offsets must have S*B+1 entries")
    if offsets[0] != 0 or np.any(np.diff(offsets) < 0) or offsets[-1] != ids.size:
        raise ValueError("invalid CSR offsets")
    lens = np.diff(offsets)
    bag = np.repeat(np.arange(S * batch, dtype=np.int64), lens)
    slot = bag // batch
    table = np.asarray(cfg.slot_table, dtype=np.int64)[slot]
    rows = np.asarray(cfg.rows, dtype=np.int64)[table]
    if np.any(ids < 0) or np.any(ids >= rows):
        raise ValueError("id out of range")
    g = cfg.base[table] + ids
    return g, bag, lens


# ----------------------------------------------------------------------------- step 3: dedup
def dedup(g: np.ndarray):
    """U = sorted unique keys, counts (multiplicities) and inverse (U[inverse[j]] == g[j]) (R5, R6)."""
    U, inverse, counts = np.unique(np.asarray(g, dtype=np.int64), return_inverse=True, return_counts=True)
    return U, counts.astype(np.int64), inverse.astype(np.int64)


# ----------------------------------------------------------------------------- step 4: routing
def owner_local(cfg: OracleConfig, g: np.ndarray):
    """R7. cyclic: owner = g mod W, local = g div W. block: rows_per = ceil(R_total / W),
    owner = g div rows_per, local = g mod rows_per."""
    g = np.asarray(g, dtype=np.int64)
    W = cfg.world
    if cfg.shard == "cyclic":
        return g % W, g // W
    rows_per = -(-cfg.total_rows // W)
    return g // rows_per, g % rows_per


def rows_local(cfg: OracleConfig, rank: int) -> int:
    W, R = cfg.world, cfg.total_rows
    if cfg.shard == "cyclic":
        return (R - rank + W - 1) // W
    rows_per = -(-R // W)
    return max(0, min(R, (rank + 1) * rows_per) - rank * rows_per)


def route(cfg: OracleConfig, U: np.ndarray):
    """Send lists r -> d = {g in U : owner(g) = d}, ascending; counts C[d] = |send list d|."""
    owner, _ = owner_local(cfg, U)
    lists = [U[owner == d] for d in range(cfg.world)]
    return lists, np.array([x.size for x in lists], dtype=np.int64)


def owner_sets(cfg: OracleConfig, per_rank_U: Sequence[np.ndarray], per_rank_counts: Sequence[np.ndarray]):
    """U_o(d) = union over ranks r of the send lists r -> d; owner count[g] = sum_r count_r[g]."""
    out = []
    for d in range(cfg.world):
        keys, cnts = [], []
        for U, c in zip(per_rank_U, per_rank_counts):
            own, _ = owner_local(cfg, U)
            keys.append(U[own == d])
            cnts.append(c[own == d])
        k = np.concatenate(keys) if keys else np.zeros(0, np.int64)
        c = np.concatenate(cnts) if cnts else np.zeros(0, np.int64)
        Uo, inv = np.unique(k, return_inverse=True)
        tot = np.zeros(Uo.size, dtype=np.int64)
        np.add.at(tot, inv, c)
        out.append((Uo, tot))
    return out


# ----------------------------------------------------------------------------- state (sparse store)
class SparseState:
    """fp32 table rows (+ Adagrad accumulator) held only for touched keys; untouched rows are
    regenerated from the R15 hash (so a 1e9-row table needs no host memory)."""

    def __init__(self, cfg: OracleConfig):
        self.cfg = cfg
        self.keys = np.zeros(0, dtype=np.int64)
        self.w = np.zeros((0, cfg.dim), dtype=np.float32)
        self.a = np.zeros((0, cfg.accum_width), dtype=np.float32)

    def _find(self, g):
        pos = np.searchsorted(self.keys, g)
        pos_c = np.minimum(pos, max(self.keys.size - 1, 0))
        hit = (self.keys.size > 0) & (self.keys[pos_c] == g) if self.keys.size else np.zeros(g.shape, bool)
        return pos_c, hit

    def get(self, g: np.ndarray):
        g = np.asarray(g, dtype=np.int64).reshape(-1)
        w = init_weights(self.cfg.seed, g, self.cfg.dim)
        a = np.full((g.size, self.cfg.accum_width), self.cfg.init_accum, dtype=np.float32)
        if self.keys.size and g.size:
            pos, hit = self._find(g)
            w[hit] = self.w[pos[hit]]
            a[hit] = self.a[pos[hit]]
        return w, a

    def set(self, g: np.ndarray, w: np.ndarray, a: np.ndarray):
        g = np.asarray(g, dtype=np.int64).reshape(-1)
        if g.size == 0:
            return
        if self.keys.size:
            pos, hit = self._find(g)
            self.w[pos[hit]] = w[hit]
            self.a[pos[hit]] = a[hit]
            new = ~hit
        else:
            new = np.ones(g.size, bool)
        if np.any(new):
            keys = np.concatenate([self.keys, g[new]])
            order = np.argsort(keys, kind="stable")
            self.keys = keys[order]
            self.w = np.concatenate([self.w, w[new]])[order]
            self.a = np.concatenate([self.a, a[new]])[order]


# ----------------------------------------------------------------------------- step 2: forward
def pool_forward(cfg: OracleConfig, state: SparseState, ids, offsets, batch: int) -> np.ndarray:
    """Y[b, s, :] = fp32(sum over the bag of W_t[id, :]) accumulated in fp64; mean divides the fp64 sum
    by the bag length counting duplicates (R1, R3); empty bag -> 0 (R2). Returns float32 [B][S][D]."""
    S, D = len(cfg.slot_table), cfg.dim
    g, bag, lens = occurrence_keys(cfg, ids, offsets, batch)
    w, _ = state.get(g)
    Y = np.zeros((S * batch, D), dtype=np.float64)
    np.add.at(Y, bag, w.astype(np.float64))
    if cfg.pool == "mean":
        nz = lens > 0
        Y[nz] /= lens[nz, None].astype(np.float64)
    return Y.reshape(S, batch, D).transpose(1, 0, 2).astype(np.float32)


# ----------------------------------------------------------------------------- step 6: backward merge
def merged_grads(cfg: OracleConfig, per_rank_batches: Sequence[Tuple[np.ndarray, np.ndarray, int, np.ndarray]]):
    """G[g] = sum over all ranks and occurrences of c_j, fp64; c_j = dY[b, s, :] (sum) or dY/|bag| (mean).
    per_rank_batches: [(ids, offsets, B, dY[B][S][D])]. Returns (touched keys sorted, G fp64 [U, D])."""
    D = cfg.dim
    all_g, all_c = [], []
    for ids, offsets, B, dy in per_rank_batches:
        g, bag, lens = occurrence_keys(cfg, ids, offsets, B)
        S = len(cfg.slot_table)
        dy_bags = np.asarray(dy, dtype=np.float32).transpose(1, 0, 2).reshape(S * B, D).astype(np.float64)
        c = dy_bags[bag]
        if cfg.pool == "mean":
            c = c / lens[bag][:, None].astype(np.float64)
        all_g.append(g)
        all_c.append(c)
    g = np.concatenate(all_g) if all_g else np.zeros(0, np.int64)
    c = np.concatenate(all_c) if all_c else np.zeros((0, D))
    U, inv = np.unique(g, return_inverse=True)
    G = np.zeros((U.size, D), dtype=np.float64)
    np.add.at(G, inv.reshape(-1), c)
    return U, G


# ----------------------------------------------------------------------------- step 7: update
def sgd_update(w: np.ndarray, G: np.ndarray, lr: float) -> np.ndarray:
    """w <- w - lr*G, fp64 from the fp32 state, one rounding."""
    return (w.astype(np.float64) - lr * G).astype(np.float32)


def adagrad_update(w: np.ndarray, a: np.ndarray, G: np.ndarray, lr: float, eps: float):
    """Element-wise Adagrad (R12): a <- a + G^2; w <- w - lr*G/(sqrt(a)+eps); fp64, one rounding each."""
    a64 = a.astype(np.float64) + G * G
    w64 = w.astype(np.float64) - lr * G / (np.sqrt(a64) + eps)
    return w64.astype(np.float32), a64.astype(np.float32)


def rowwise_adagrad_update(w: np.ndarray, a: np.ndarray, G: np.ndarray, lr: float, eps: float):
    """Row-wise Adagrad (reading R14'): one accumulator per row, a [U, 1]:
    a <- a + (1/D) sum_c G[c]^2;  w <- w - lr*G/(sqrt(a)+eps); fp64, one rounding each."""
    a64 = a.astype(np.float64) + np.mean(G * G, axis=1, keepdims=True)
    w64 = w.astype(np.float64) - lr * G / (np.sqrt(a64) + eps)
    return w64.astype(np.float32), a64.astype(np.float32)


def apply_update(cfg: OracleConfig, state: SparseState, U: np.ndarray, G: np.ndarray, lr: float):
    w, a = state.get(U)
    if cfg.opt == "sgd":
        state.set(U, sgd_update(w, G, lr), a)
    elif cfg.opt == "rowwise_adagrad":
        w2, a2 = rowwise_adagrad_update(w, a, G, lr, cfg.eps)
        state.set(U, w2, a2)
    else:
        w2, a2 = adagrad_update(w, a, G, lr, cfg.eps)
        state.set(U, w2, a2)


# ----------------------------------------------------------------------------- whole step (W logical ranks)
class OracleEmbedding:
    """Synchronous W-rank semantics run serially in one process (SPEC idea S:484): every rank's lookup
    reads the pre-step state; one merged update per touched row per step (R9); step k+1 reads the
    updated rows (synchronous executor)."""

    def __init__(self, cfg: OracleConfig):
        self.cfg = cfg
        self.state = SparseState(cfg)
        self._pending = None

    def lookup(self, per_rank: Sequence[Tuple[np.ndarray, np.ndarray, int]]) -> List[np.ndarray]:
        self._pending = [(np.asarray(i), np.asarray(o), int(B)) for i, o, B in per_rank]
        return [pool_forward(self.cfg, self.state, i, o, B) for i, o, B in self._pending]

    def backward_update(self, per_rank_dy: Sequence[np.ndarray], lr: float):
        if self._pending is None:
            raise RuntimeError("backward_update without lookup")
        U, G = merged_grads(self.cfg, [(i, o, B, dy) for (i, o, B), dy in zip(self._pending, per_rank_dy)])
        apply_update(self.cfg, self.state, U, G, lr)
        self._pending = None
        return U

    def rows(self, g: np.ndarray):
        return self.state.get(g)

    def load_rows(self, g: np.ndarray, w: np.ndarray, a: np.ndarray):
        """Stepwise-resync protocol (R22): load another implementation's pre-step state for rows g."""
        self.state.set(np.asarray(g, dtype=np.int64), np.asarray(w, np.float32), np.asarray(a, np.float32))

    # per-rank bit-exact pieces ------------------------------------------------
    def rank_dedup_route(self, ids, offsets, B):
        g, _, _ = occurrence_keys(self.cfg, ids, offsets, B)
        U, counts, inverse = dedup(g)
        lists, send_counts = route(self.cfg, U)
        return U, counts, inverse, lists, send_counts
