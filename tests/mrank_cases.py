"""Row-sharded (W > 1) parity cases shared by the group-mode test (all ranks in one process, any number
of GPUs: tests/test_group_parity.py) and the one-process-per-GPU worker (tests/mgpu_worker.py).

Per step (stepwise-resynced protocol R22): every rank's owned touched rows are read from the GPU and
loaded into the serial oracle, then the layer's Y per rank (tolerance R21), the per-rank dedup and
per-owner send counts (bit-exact), the owner-side distinct rows and their fan-in (bit-exact), the
receive counts (consistent with the senders') and every updated owned row are compared with the
single-process oracle run on all ranks' batches (SPEC idea "distributed == serial, fixed
rank order").
"""
import numpy as np

import synthgen
from oracle import emb_oracle as O

RTOL, ATOL = 1e-5, 1e-6


def close(a, b):
    return bool(np.all(np.abs(a.astype(np.float64) - b.astype(np.float64)) <= ATOL + RTOL * np.abs(b)))


def case_workload(case, world):
    """(workload, per-rank batch, steps) of a named case."""
    if case in ("c3", "c3rw", "c3full"):
        wl = synthgen.WORKLOADS["C3"]
        if case == "c3rw":  # row-wise Adagrad
            wl = wl.with_(opt="rowwise_adagrad", init_accum=0.1)
        B = wl.batch - 16 * (world - 1) if case == "c3full" else 2048  # c3full: BJ:9 per-GPU batch
        return wl, B, (2 if case == "c3full" else 3)
    if case == "edge":  # ranks with no ids: batch 0 (rank 1, step 1), all bags empty (rank 0, step 2)
        wl = synthgen.WORKLOADS["C3"].with_(rows=(40_000, 30_000, 20_000), slot_table=(0, 1, 2), pool="mean")
        return wl, 512, 3
    if case == "gen":  # non-monotone slot -> table map: key kernel + general radix sort
        wl = synthgen.WORKLOADS["C1"].with_(rows=(50_000, 30_000), slot_table=(1, 0, 1), ids="zipf", zipf_s=1.1,
                                            opt="adagrad", pool="mean")
        return wl, 512, 3
    if case == "hot":  # hot ids (C5 structure, bag 8), mean pooling, SGD
        wl = synthgen.WORKLOADS["C5"].with_(bag_len=8, pool="mean", opt="sgd")
        return wl, 256, 3
    if case == "skew":  # a 5-row table: one sort range of > 8,192 ids (shared-memory cap) -> global-scratch path
        wl = synthgen.WORKLOADS["C3"].with_(rows=(5, 60_000), slot_table=(0, 1), dim=16)
        return wl, 10_000, 2
    if case == "c5":  # C5 exactly (bag 64, 90% of ids in the per-table top 1000), reduced batch
        wl = synthgen.WORKLOADS["C5"]
        return wl, 256, 2
    raise ValueError(case)


def case_batch(case, wl, B, rank, step):
    if case == "edge" and step == 1 and rank == 1:
        return synthgen.make_batch(wl, rank=rank, step=step, batch=0)
    if case == "edge" and step == 2 and rank == 0:
        return synthgen.make_batch(wl, rank=rank, step=step, batch=B, empty_frac=1.0)
    return synthgen.make_batch(wl, rank=rank, step=step, batch=B + 16 * rank)


def owned_touched(cfg1, cfgW, batches, rank):
    """Fused keys touched by any rank's batch that `rank` owns, and their table index."""
    touched = np.unique(np.concatenate([O.occurrence_keys(cfg1, b.ids, b.offsets, b.batch)[0] for b in batches]))
    own, _ = O.owner_local(cfgW, touched)
    mine = touched[own == rank]
    return mine, np.searchsorted(cfg1.base, mine, side="right") - 1


def read_owned(layer, cfg1, mine, t_of, dim):
    w = np.empty((mine.size, dim), np.float32)
    a = np.empty((mine.size, layer.accum_width), np.float32)
    for t in np.unique(t_of):
        m = t_of == t
        w[m], a[m] = layer.read_rows(int(t), mine[m] - cfg1.base[t])
    return w, a


def check_rank_step(msgs, s, rank, cfgW, ora, batches, Y, Yo, info, keys, counts, okeys, fanin, recv_counts_expected):
    """Forward-side checks of one rank after its lookup (returns nothing; appends failures to msgs)."""
    if not close(Y, Yo):
        msgs.append(f"step {s} rank {rank}: Y mismatch (max err {np.abs(Y - Yo).max():.3g})")
    bt = batches[rank]
    Ur, cr, _, _, _ = ora.rank_dedup_route(bt.ids, bt.offsets, bt.batch)
    _, sc = O.route(cfgW, Ur)
    if not (np.array_equal(keys.astype(np.int64), Ur) and np.array_equal(counts, cr)):
        msgs.append(f"step {s} rank {rank}: unique/counts differ")
    if list(info["send_counts"]) != sc.tolist():
        msgs.append(f"step {s} rank {rank}: send counts {info['send_counts']} vs {sc.tolist()}")
    per_U = [ora.rank_dedup_route(b.ids, b.offsets, b.batch) for b in batches]
    osets = O.owner_sets(cfgW, [p[0] for p in per_U], [p[1] for p in per_U])
    if not np.array_equal(okeys.astype(np.int64), osets[rank][0]):
        msgs.append(f"step {s} rank {rank}: owner unique set differs ({okeys.size} vs {osets[rank][0].size})")
    exp_fanin = sum(np.isin(osets[rank][0], p[0]).astype(np.int64) for p in per_U)
    if not np.array_equal(fanin, exp_fanin):
        msgs.append(f"step {s} rank {rank}: owner fan-in differs")
    if info["recv_counts"] != recv_counts_expected:
        msgs.append(f"step {s} rank {rank}: recv counts {info['recv_counts']} vs senders' {recv_counts_expected}")
    if info["unique_owner"] != osets[rank][0].size:
        msgs.append(f"step {s} rank {rank}: unique_owner {info['unique_owner']} vs {osets[rank][0].size}")
