#!/usr/bin/env python
"""Per-kernel timing of the W > 1 step in group mode (all ranks in this process): the same kernels a
one-process-per-GPU rank runs, on one GPU (ranks emulated, --devices same) or one GPU per rank
(--devices distinct, peer access). Used for ncu captures of the exchange kernels on a single GPU
(ncu must not wrap a multi-rank command).

  python tools/group_bench.py --world 2 --devices same --steps 20 [--workload C3] [--batch B]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synthgen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--devices", choices=["same", "distinct"], default="same")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--profile", action="store_true", help="per-kernel CUDA events (libemb profiler)")
    args = ap.parse_args()
    import torch
    from paper_2112_02752_b200.harness import DeviceBatch, make_group
    W = args.world
    wl = synthgen.WORKLOADS[args.workload]
    if args.batch:
        wl = wl.with_(batch=args.batch)
    devices = list(range(W)) if args.devices == "distinct" else [0] * W
    bts = [[synthgen.make_batch(wl, rank=r, step=s) for r in range(W)] for s in range(4)]
    grp = make_group(wl, world=W, max_batch=wl.batch, max_ids=max(b.nnz for st in bts for b in st), devices=devices)
    dbs = [[DeviceBatch(b, wl.num_slots, wl.dim, devices[r]) for r, b in enumerate(st)] for st in bts]
    streams = [torch.cuda.current_stream(d) for d in devices]

    def step(i):
        db = dbs[i % len(dbs)]
        grp.lookup([d.ids for d in db], [d.offsets for d in db], [d.batch for d in db], [d.nnz for d in db],
                   [d.out for d in db], streams)
        grp.backward_update([d.dy for d in db], wl.lr, streams)

    for i in range(args.warmup):
        step(i)
    for d in set(devices):
        torch.cuda.synchronize(d)
    if args.profile:
        for lay in grp.layers:
            lay.profile(True)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(streams[0])
    for i in range(args.steps):
        step(i)
    for r in range(W):
        if devices[r] != devices[0]:
            e = torch.cuda.Event()
            e.record(streams[r])
            streams[0].wait_event(e)
    ev1.record(streams[0])
    for d in set(devices):
        torch.cuda.synchronize(d)
    out = {"world": W, "devices": args.devices, "workload": wl.name, "ms_per_step": ev0.elapsed_time(ev1) / args.steps}
    if args.profile:
        per = [lay.profile_read() for lay in grp.layers]
        out["kernels_us_per_launch"] = {k: [round(1e3 * p[k][0] / max(p[k][1], 1), 2) if k in p else None for p in per]
                                        for k in sorted(set().union(*per))}
    print(json.dumps(out))
    grp.close()


if __name__ == "__main__":
    main()
