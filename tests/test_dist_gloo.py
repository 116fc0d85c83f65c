"""World-size-2 and -8 CPU tests (gloo) of the N>1 host logic (-m "not gpu"):
  * the ncclUniqueId broadcast and the max-over-ranks timing reduction of paper_2112_02752_b200.dist;
  * the row-sharded exchange protocol that libemb implements with its peer-memory kernels (DESIGN.md
    §8), replayed with torch.distributed all-to-alls and oracle arithmetic per rank: per-rank dedup ->
    per-owner ascending key lists + counts (libemb: the route, KEYS) -> keys to owners -> the owners'
    rows back (libemb: gather-push, ROWS) -> pool -> per-unique-key gradients to owners (libemb: the
    requester merge, GRADS) -> source-rank-order merge -> update. Its result must equal the
    single-process oracle on the same per-rank batches (SPEC idea "distributed ==
    serial").
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthgen
from oracle import emb_oracle as O

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _a2av(send_chunks):
    """all-to-allv of per-destination int64/float64 numpy chunks (flattened), returns received chunks."""
    counts = torch.tensor([c.size for c in send_chunks], dtype=torch.int64)
    rcounts = torch.empty_like(counts)
    dist.all_to_all_single(rcounts, counts)
    dtype = send_chunks[0].dtype
    tdt = torch.float64 if dtype == np.float64 else torch.int64
    flat = torch.from_numpy(np.concatenate(send_chunks).astype(dtype)) if counts.sum() else torch.zeros(0, dtype=tdt)
    out = torch.empty(int(rcounts.sum()), dtype=tdt)
    dist.all_to_all_single(out, flat.to(tdt), rcounts.tolist(), counts.tolist())
    res, o = [], 0
    for c in rcounts.tolist():
        res.append(out[o:o + c].numpy())
        o += c
    return res


def _worker(rank, W, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=W)
        from paper_2112_02752_b200 import dist as D
        uid = D.share_unique_id(lambda: bytes(range(128)))
        assert uid == bytes(range(128))
        assert D.max_over_ranks(float(rank) + 0.5) == W - 0.5

        wl = synthgen.WORKLOADS["C3"].with_(rows=(5000, 3000, 700), slot_table=(0, 1, 2), dim=8, ids="zipf",
                                            zipf_s=1.1, batch=64)
        cfgW = O.config_from_workload(wl, world=W)
        D_ = wl.dim
        # owner shard (oracle rows of the keys this rank owns)
        shard = O.SparseState(cfgW)
        ok = True
        for step in range(2):
            bt = synthgen.make_batch(wl, rank=rank, step=step, batch=64 + 8 * rank)
            g, bag, lens = O.occurrence_keys(cfgW, bt.ids, bt.offsets, bt.batch)
            U, counts, inv = O.dedup(g)
            lists, send_counts = O.route(cfgW, U)
            # X1: keys to owners (owner-major send order, ascending inside an owner)
            recv_keys = _a2av([lst.astype(np.int64) for lst in lists])
            # owner gathers its rows (from its shard state) and X2 returns them
            rows_back = [shard.get(rk)[0].astype(np.float64).reshape(-1) for rk in recv_keys]
            got = _a2av(rows_back)
            uniq_rows = np.zeros((U.size, D_))
            order = np.concatenate(lists) if U.size else np.zeros(0, np.int64)
            pos = np.searchsorted(U, order)
            uniq_rows[pos] = np.concatenate(got).reshape(-1, D_) if U.size else uniq_rows
            # pool from the received unique rows
            Y = np.zeros((wl.num_slots * bt.batch, D_))
            np.add.at(Y, bag, uniq_rows[inv])
            Y = Y.reshape(wl.num_slots, bt.batch, D_).transpose(1, 0, 2).astype(np.float32)
            # reference: single-process oracle on all ranks' batches (serial), then compare this rank's Y
            ref = O.OracleEmbedding(O.config_from_workload(wl, world=1))
            all_bt = [synthgen.make_batch(wl, rank=r, step=s, batch=64 + 8 * r) for s in range(step + 1)
                      for r in range(W)]
            for s in range(step):
                ref.lookup([(b.ids, b.offsets, b.batch) for b in all_bt[s * W:(s + 1) * W]])
                ref.backward_update([b.dy for b in all_bt[s * W:(s + 1) * W]], 0.05)
            Yref = ref.lookup([(b.ids, b.offsets, b.batch) for b in all_bt[step * W:(step + 1) * W]])[rank]
            ok &= bool(np.array_equal(Y, Yref))
            # backward: per-unique-key local gradient in fp64, X3 to owners, source-order merge, update
            c = bt.dy.transpose(1, 0, 2).reshape(-1, D_).astype(np.float64)[bag]
            gloc = np.zeros((U.size, D_))
            np.add.at(gloc, inv, c)
            send = [gloc[np.searchsorted(U, lst)].reshape(-1) for lst in lists]
            grecv = _a2av(send)
            keys_all = np.concatenate(recv_keys)
            g_all = np.concatenate([x.reshape(-1, D_) for x in grecv]) if keys_all.size else np.zeros((0, D_))
            Uo, oinv = np.unique(keys_all, return_inverse=True)
            G = np.zeros((Uo.size, D_))
            np.add.at(G, oinv, g_all)  # source-rank order (concatenation order)
            O.apply_update(cfgW, shard, Uo, G, 0.05)
            ref.backward_update([b.dy for b in all_bt[step * W:(step + 1) * W]], 0.05)
            if Uo.size:
                ok &= bool(np.allclose(shard.get(Uo)[0], ref.rows(Uo)[0], rtol=1e-6, atol=1e-7))
                own, _ = O.owner_local(cfgW, Uo)
                ok &= bool(np.all(own == rank))
        q.put((rank, ok, None))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, False, traceback.format_exc()))


@pytest.mark.timeout(600)
@pytest.mark.parametrize("W", [2, 8])
def test_exchange_protocol_equals_serial(W):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, W, port, q)) for r in range(W)]
    for p in ps:
        p.start()
    res = [q.get(timeout=560) for _ in range(W)]
    for p in ps:
        p.join(timeout=60)
    for rank, ok, err in res:
        assert err is None, err
        assert ok, f"rank {rank} diverged from the serial oracle"
