"""Per-rank body of the multi-GPU parity test (launched by tests/test_multigpu.py through torchrun, one
process per GPU). Row-sharded layer over W GPUs (NCCL exchanges inside libemb) vs the serial CPU oracle
on the same per-rank batches: Y per rank, routing counts (bit-exact), owner-side unique rows
(bit-exact), and every updated owned row after each step (stepwise tolerance R21).
Exit code 0 = pass."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synthgen  # noqa: E402
from oracle import emb_oracle as O  # noqa: E402
from paper_2112_02752_b200 import dist as D  # noqa: E402
from paper_2112_02752_b200 import emb as E  # noqa: E402
from paper_2112_02752_b200.harness import DeviceBatch, make_layer  # noqa: E402

RTOL, ATOL = 1e-5, 1e-6


def close(a, b):
    return bool(np.all(np.abs(a.astype(np.float64) - b.astype(np.float64)) <= ATOL + RTOL * np.abs(b)))


def main():
    rank, world, local = D.env_rank()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nid = D.share_unique_id(E.get_unique_id)
    case = os.environ.get("EMB_MGPU_CASE", "c3")
    shard = os.environ.get("EMB_MGPU_SHARD", "cyclic")
    if case in ("c3", "c3rw", "c3full"):
        wl = synthgen.WORKLOADS["C3"]
        if case == "c3rw":  # row-wise Adagrad
            wl = wl.with_(opt="rowwise_adagrad", init_accum=0.1)
        B = wl.batch - 16 * (world - 1) if case == "c3full" else 2048  # c3full: BJ:9 per-GPU batch
    elif case == "edge":  # ranks with no ids: batch 0 (rank 1, step 1), all bags empty (rank 0, step 2)
        wl = synthgen.WORKLOADS["C3"].with_(rows=(40_000, 30_000, 20_000), slot_table=(0, 1, 2), pool="mean")
        B = 512
    elif case == "gen":  # non-monotone slot -> table map: key kernel + general radix sort + NCCL exchange
        wl = synthgen.WORKLOADS["C1"].with_(rows=(50_000, 30_000), slot_table=(1, 0, 1), ids="zipf", zipf_s=1.1,
                                            opt="adagrad", pool="mean")
        B = 512
    else:  # hot ids, mean pooling, sgd
        wl = synthgen.WORKLOADS["C5"].with_(bag_len=8, pool="mean", opt="sgd")
        B = 256
    cfgW = O.config_from_workload(wl, world=world, shard=shard)
    cfg1 = O.config_from_workload(wl, world=1)
    steps = 2 if case == "c3full" else 3
    def _batch(r, s_):
        if case == "edge" and s_ == 1 and r == 1:
            return synthgen.make_batch(wl, rank=r, step=s_, batch=0)
        if case == "edge" and s_ == 2 and r == 0:
            return synthgen.make_batch(wl, rank=r, step=s_, batch=B, empty_frac=1.0)
        return synthgen.make_batch(wl, rank=r, step=s_, batch=B + 16 * r)

    bts = [[_batch(r, s) for r in range(world)] for s in range(steps)]
    layer = make_layer(wl, max_batch=B + 16 * world, max_ids=max(b.nnz for st in bts for b in st), world=world,
                       rank=rank, nccl_id=nid, device=local, shard=shard)
    ora = O.OracleEmbedding(cfg1)
    ok = True
    msgs = []
    for s in range(steps):
        batch_list = bts[s]
        # stepwise resync (R22): load this rank's owned touched rows into the oracle ... from every rank
        touched = np.unique(np.concatenate([O.occurrence_keys(cfg1, b.ids, b.offsets, b.batch)[0]
                                            for b in batch_list]))
        own, _ = O.owner_local(cfgW, touched)
        mine = touched[own == rank]
        t_of = np.searchsorted(cfg1.base, mine, side="right") - 1
        w_mine = np.empty((mine.size, wl.dim), np.float32)
        a_mine = np.empty((mine.size, layer.accum_width), np.float32)
        for t in np.unique(t_of):
            m = t_of == t
            w_mine[m], a_mine[m] = layer.read_rows(int(t), mine[m] - cfg1.base[t])
        # share pre-step rows so every rank's oracle has the GPU state of all touched rows
        gathered = [None] * world
        dist.all_gather_object(gathered, (mine, w_mine, a_mine))
        for gk, gw_, ga in gathered:
            if gk.size:
                ora.load_rows(gk, gw_, ga)
        bt = batch_list[rank]
        db = DeviceBatch(bt, wl.num_slots, wl.dim, local)
        layer.lookup(db.ids, db.offsets, db.batch, db.nnz, db.out)
        torch.cuda.synchronize()
        Y = db.out.cpu().numpy()
        info = layer.step_info()
        keys, counts = layer.last_unique()
        okeys, fanin = layer.last_owner_unique()
        Yo = ora.lookup([(b.ids, b.offsets, b.batch) for b in batch_list])[rank]
        if not close(Y, Yo):
            ok = False
            msgs.append(f"step {s}: Y mismatch (max err {np.abs(Y - Yo).max():.3g})")
        Ur, cr, _, _, _ = ora.rank_dedup_route(bt.ids, bt.offsets, bt.batch)
        _, sc = O.route(cfgW, Ur)
        if not (np.array_equal(keys.astype(np.int64), Ur) and np.array_equal(counts, cr)):
            ok = False
            msgs.append(f"step {s}: unique/counts differ")
        if list(info["send_counts"]) != sc.tolist():
            ok = False
            msgs.append(f"step {s}: send counts {info['send_counts']} vs {sc.tolist()}")
        per_U = [ora.rank_dedup_route(b.ids, b.offsets, b.batch) for b in batch_list]
        osets = O.owner_sets(cfgW, [p[0] for p in per_U], [p[1] for p in per_U])
        if not np.array_equal(okeys.astype(np.int64), osets[rank][0]):
            ok = False
            msgs.append(f"step {s}: owner unique set differs ({okeys.size} vs {osets[rank][0].size})")
        exp_fanin = sum(np.isin(osets[rank][0], p[0]).astype(np.int64) for p in per_U)
        if not np.array_equal(fanin, exp_fanin):
            ok = False
            msgs.append(f"step {s}: owner fan-in differs")
        recv = [None] * world
        dist.all_gather_object(recv, info["send_counts"])
        if info["recv_counts"] != [recv[r][rank] for r in range(world)]:
            ok = False
            msgs.append(f"step {s}: recv counts inconsistent")
        if case == "c3":  # emb_lookup_prefetch is a documented no-op at W > 1: results must not change
            layer.lookup_prefetch(db.ids, db.offsets, db.batch, db.nnz)
        layer.backward_update(db.dy, wl.lr)
        torch.cuda.synchronize()
        ora.backward_update([b.dy for b in batch_list], wl.lr)
        w_after = np.empty_like(w_mine)
        a_after = np.empty_like(a_mine)
        for t in np.unique(t_of):
            m = t_of == t
            w_after[m], a_after[m] = layer.read_rows(int(t), mine[m] - cfg1.base[t])
        wo, ao = ora.rows(mine)
        if not close(w_after, wo):
            ok = False
            msgs.append(f"step {s}: updated w mismatch (max err {np.abs(w_after - wo).max():.3g})")
        if wl.opt != "sgd" and not close(a_after, ao):
            ok = False
            msgs.append(f"step {s}: updated a mismatch")
    layer.close()
    res = [None] * world
    dist.all_gather_object(res, (ok, msgs))
    dist.destroy_process_group()
    if rank == 0:
        for r, (o, m) in enumerate(res):
            print(f"rank {r}: {'ok' if o else 'FAIL'} {m}")
    sys.exit(0 if all(o for o, _ in res) else 1)


if __name__ == "__main__":
    main()
