"""Per-rank body of the one-process-per-GPU parity test (launched by tests/test_multigpu.py through
torchrun): the row-sharded layer over W GPUs (libemb's peer-memory exchange between processes, CUDA IPC
mappings bootstrapped over NCCL) vs the serial CPU oracle on the same per-rank batches. Checks per step:
tests/mrank_cases.py. Exit code 0 = pass."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import emb_oracle as O  # noqa: E402
from paper_2112_02752_b200 import dist as D  # noqa: E402
from paper_2112_02752_b200 import emb as E  # noqa: E402
from paper_2112_02752_b200.harness import DeviceBatch, make_layer  # noqa: E402
import mrank_cases as C  # noqa: E402


def main():
    rank, world, local = D.env_rank()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nid = D.share_unique_id(E.get_unique_id)
    case = os.environ.get("EMB_MGPU_CASE", "c3")
    shard = os.environ.get("EMB_MGPU_SHARD", "cyclic")
    # EMB_MGPU_PREFETCH=1: the next step's first phase (sort + route) is prefetched before each backward
    prefetch = os.environ.get("EMB_MGPU_PREFETCH", "0") == "1"
    wl, B, steps = C.case_workload(case, world)
    cfgW = O.config_from_workload(wl, world=world, shard=shard)
    cfg1 = O.config_from_workload(wl, world=1)
    bts = [[C.case_batch(case, wl, B, r, s) for r in range(world)] for s in range(steps)]
    layer = make_layer(wl, max_batch=B + 16 * world, max_ids=max(max(b.nnz for st in bts for b in st), 1),
                       world=world, rank=rank, nccl_id=nid, device=local, shard=shard)
    ora = O.OracleEmbedding(cfg1)
    msgs = []
    dbs = [DeviceBatch(bts[s][rank], wl.num_slots, wl.dim, local) for s in range(steps)]
    for s in range(steps):
        batches = bts[s]
        mine, t_of = C.owned_touched(cfg1, cfgW, batches, rank)
        w_mine, a_mine = C.read_owned(layer, cfg1, mine, t_of, wl.dim)
        gathered = [None] * world  # stepwise resync (R22): every rank's oracle gets all touched rows
        dist.all_gather_object(gathered, (mine, w_mine, a_mine))
        for gk, gw_, ga in gathered:
            if gk.size:
                ora.load_rows(gk, gw_, ga)
        db = dbs[s]
        layer.lookup(db.ids, db.offsets, db.batch, db.nnz, db.out)
        torch.cuda.synchronize()
        info = layer.step_info()
        keys, counts = layer.last_unique()
        okeys, fanin = layer.last_owner_unique()
        Yo = ora.lookup([(b.ids, b.offsets, b.batch) for b in batches])[rank]
        sends = [None] * world
        dist.all_gather_object(sends, info["send_counts"])
        C.check_rank_step(msgs, s, rank, cfgW, ora, batches, db.out.cpu().numpy(), Yo, info, keys, counts, okeys,
                          fanin, [sends[q][rank] for q in range(world)])
        if prefetch and s + 1 < steps:
            nx = dbs[s + 1]
            layer.lookup_prefetch(nx.ids, nx.offsets, nx.batch, nx.nnz)
        layer.backward_update(db.dy, wl.lr)
        torch.cuda.synchronize()
        ora.backward_update([b.dy for b in batches], wl.lr)
        w_after, a_after = C.read_owned(layer, cfg1, mine, t_of, wl.dim)
        wo, ao = ora.rows(mine)
        if not C.close(w_after, wo):
            msgs.append(f"step {s}: updated w mismatch (max err {np.abs(w_after - wo).max():.3g})")
        if wl.opt != "sgd" and not C.close(a_after, ao):
            msgs.append(f"step {s}: updated a mismatch")
    layer.close()
    res = [None] * world
    dist.all_gather_object(res, (not msgs, msgs))
    dist.destroy_process_group()
    if rank == 0:
        for r, (o, m) in enumerate(res):
            print(f"rank {r}: {'ok' if o else 'FAIL'} {m}")
    sys.exit(0 if all(o for o, _ in res) else 1)


if __name__ == "__main__":
    main()
