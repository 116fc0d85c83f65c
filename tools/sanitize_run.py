#!/usr/bin/env python
"""Small end-to-end run of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per gpurun call): C1 at W = 1 (sort path, SGD, mean pooling), a general-sort-path
layer (non-monotone slot map, Adagrad), row-wise Adagrad, and a W = 2 group (both ranks on cuda:0:
route, merge tree, gather-push, requester and owner gradient passes). Checks every output against the
CPU oracle so a sanitizer-clean run is also a correct one.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synthgen  # noqa: E402
from oracle import emb_oracle as O  # noqa: E402


def close(a, b):
    return bool(np.all(np.abs(a.astype(np.float64) - b.astype(np.float64)) <= 1e-6 + 1e-5 * np.abs(b)))


def w1_case(torch, wl, B, steps=2):
    from paper_2112_02752_b200.harness import DeviceBatch, make_layer
    cfg = O.config_from_workload(wl)
    bts = [synthgen.make_batch(wl, step=k, batch=B) for k in range(steps)]
    layer = make_layer(wl, max_batch=B, max_ids=max(b.nnz for b in bts))
    ora = O.OracleEmbedding(cfg)
    ok = True
    for bt in bts:
        db = DeviceBatch(bt, wl.num_slots, wl.dim, 0)
        layer.lookup(db.ids, db.offsets, db.batch, db.nnz, db.out)
        layer.backward_update(db.dy, wl.lr)
        torch.cuda.synchronize()
        (Yo,) = ora.lookup([(bt.ids, bt.offsets, bt.batch)])
        ora.backward_update([bt.dy], wl.lr)
        ok &= close(db.out.cpu().numpy(), Yo)
    layer.close()
    return ok


def group_case(torch, W=2, B=256):
    from paper_2112_02752_b200.harness import DeviceBatch, make_group
    wl = synthgen.WORKLOADS["C3"].with_(rows=(40_000, 30_000, 20_000), slot_table=(0, 1, 2), dim=16)
    cfg = O.config_from_workload(wl)
    bts = [[synthgen.make_batch(wl, rank=r, step=s, batch=B) for r in range(W)] for s in range(2)]
    grp = make_group(wl, world=W, max_batch=B, max_ids=max(b.nnz for st in bts for b in st))
    ora = O.OracleEmbedding(cfg)
    ok = True
    for st in bts:
        dbs = [DeviceBatch(b, wl.num_slots, wl.dim, 0) for b in st]
        grp.lookup([d.ids for d in dbs], [d.offsets for d in dbs], [d.batch for d in dbs], [d.nnz for d in dbs],
                   [d.out for d in dbs])
        grp.backward_update([d.dy for d in dbs], wl.lr)
        torch.cuda.synchronize()
        Yo = ora.lookup([(b.ids, b.offsets, b.batch) for b in st])
        ora.backward_update([b.dy for b in st], wl.lr)
        ok &= all(close(d.out.cpu().numpy(), y) for d, y in zip(dbs, Yo))
    grp.close()
    return ok


def main():
    import torch
    res = {
        "c1_sgd_mean": w1_case(torch, synthgen.WORKLOADS["C1"].with_(pool="mean"), 512),
        "general_path_adagrad": w1_case(torch, synthgen.WORKLOADS["C1"].with_(
            rows=(50_000, 30_000), slot_table=(1, 0, 1), ids="zipf", zipf_s=1.1, opt="adagrad"), 256),
        "rowwise_adagrad": w1_case(torch, synthgen.WORKLOADS["C1"].with_(
            opt="rowwise_adagrad", ids="zipf", zipf_s=1.2, dim=64), 256),
        "group_w2": group_case(torch),
    }
    print(res)
    sys.exit(0 if all(res.values()) else 1)


if __name__ == "__main__":
    main()
