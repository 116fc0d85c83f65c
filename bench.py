#!/usr/bin/env python
"""Benchmark of the sparse embedding layer step (forward lookup + backward merge + sparse Adagrad
update) through the C-ABI library, on synthetic BASELINE.json workloads.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1 : workload C2 (BJ:8, the config BASELINE's metric is quoted on): 26 slots x 10M rows/table,
        D = 64, B = 16,384, Zipf(1.05) ids, element-wise Adagrad, sum pooling. The line also carries
        `c3_w1`: C3 on this one GPU, the same-config denominator of the N > 1 (weak-scaling) lines.
N > 1 : workload C3 (BJ:9) row-sharded (cyclic) over N GPUs, B = 16,384 per GPU (weak scaling),
        launched with torchrun (one process per GPU; libemb exchanges keys / rows / gradients over
        NVLink peer memory with its own kernels); the line carries `nvlink` (bytes and link fraction).
--impl reference: the CPU oracle (oracle/, NumPy fp64) timed on the host cores on a bounded sample of
        the same workload (rank 0 only).

Prints ONE JSON line on rank 0 (see DESIGN.md §7 for every field).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synthgen  # noqa: E402

METRIC = "embedding lookups/sec and fwd+bwd+update samples/sec; % of HBM roofline"
POOL_BATCHES = 16  # distinct staged batches cycled through the timed loop (16 x ~116 MB > 126 MB L2)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy_ r+w)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def _traffic(kernel: str, opt: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` (for this optimizer) from the
    committed ncu capture, or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r02_traffic.json")))
        return d[f"{kernel}/{opt}"]["traffic_bytes"]
    except Exception:
        return None


def workload_for(n_gpus: int):
    wl = synthgen.WORKLOADS["C2"] if n_gpus == 1 else synthgen.WORKLOADS["C3"]
    return wl


def describe(wl, n):
    return (f"{wl.name}: {wl.num_slots} slots -> {wl.num_tables} tables, {wl.total_rows:,} rows total, D={wl.dim}, "
            f"B={wl.batch}/GPU, bag={'U{1..8}' if wl.bag == 'u1_8' else wl.bag_len}, ids={wl.ids}"
            f"{'(' + str(wl.zipf_s) + ')' if wl.ids == 'zipf' else ''}, {wl.opt}, {wl.pool} pool, "
            f"{'row-sharded cyclic over ' + str(n) + ' GPUs' if n > 1 else '1 GPU'}")


# ------------------------------------------------------------------------------ algorithmic bytes
def step_bytes(wl, N, SB, U_l, U_o, W):
    """HBM bytes the method must move per GPU per step."""
    D = wl.dim
    fwd = 8 * N + 8 * (SB + 1) + 4 * D * U_o + 4 * D * SB
    bwd = 4 * D * SB + 8 * N + 8 * (SB + 1) + state_bytes(wl, U_o)
    return fwd + bwd


def state_bytes(wl, U):
    """Optimizer read-modify-write per touched row: w (+ a) read and written."""
    D = wl.dim
    if wl.opt == "adagrad":
        return 16 * D * U
    if wl.opt == "rowwise_adagrad":
        return (8 * D + 8) * U
    return 8 * D * U


def kernel_bytes(name, wl, N, SB, U, W, U_l=None):
    """Algorithmic bytes of one launch of the named kernel. U = distinct rows updated by
    this GPU (U_o), U_l = distinct keys this GPU requested."""
    D = wl.dim
    U_l = U if U_l is None else U_l
    rem = U_l * (W - 1) / W  # requested keys owned by other ranks (uniform owners)
    if name == "grad_push":
        # W > 1 requester merge: dY row + sorted key/payload/dY-row index + rank per occurrence, one merged
        # double-float row (hi + lo) per requested key written (to its owner, (W-1)/W of them over NVLink)
        return 4 * D * N + 16 * N + 8 * D * U_l
    if name == "gather_push":
        # per key another rank requested from this owner: its local id + the table row read + the row
        # stored into the requester's region (over NVLink)
        return rem * (4 + 8 * D)
    if name == "grad_apply":
        if W == 1:  # dY row per occurrence + sorted key/payload/bag index per occurrence + state RMW per row
            return 4 * D * N + 12 * N + state_bytes(wl, U)
        # owner: merged key + receive position + hi/lo rows per received key (~U_l per rank) + state RMW
        return U_l * (8 + 8 * D) + state_bytes(wl, U)
    if name == "pool":
        # offsets + ids + one row per distinct key + Y write
        return 8 * (SB + 1) + 8 * N + 4 * D * U + 4 * D * SB
    return None


def nvlink_bytes(wl, U_l, W, lo_frac=1.0):
    """Bytes one GPU sends (= receives, symmetric) over NVLink per step (SURVEY §8(d) with the
    double-float gradient, reading R11''): per remote distinct key its 4-B key, its 4D-byte row back and
    its 4D-byte gradient hi half, plus the 4D-byte lo half for the fraction `lo_frac` of keys the owner
    receives from more than one rank."""
    return 0 if W == 1 else (W - 1) / W * U_l * (4 + 8 * wl.dim + 4 * wl.dim * lo_frac)


# ------------------------------------------------------------------------------ clocks sampler
class ClockSampler:
    def __init__(self, device):
        self.samples, self.reasons, self.max_mhz, self._stop = [], set(), None, threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)

    def _run(self):
        nv = self.nv
        names = {getattr(nv, n): n for n in dir(nv) if n.startswith("nvmlClocksEventReason") or
                 n.startswith("nvmlClocksThrottleReason")}
        bits = {
            "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4, "gpu_idle": 0x1,
            "applications_clocks_setting": 0x2, "sync_boost": 0x10, "display_clock_setting": 0x100,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h) if hasattr(
                    nv, "nvmlDeviceGetCurrentClocksEventReasons") else nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for n, b in bits.items():
                    if r & b and n != "gpu_idle":
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "nvml unavailable"}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------ CPU oracle timing
def oracle_time(wl, budget_s=15.0, max_steps=None, batch=None):
    """Time the oracle (as it stands) on host cores: full steps (lookup + backward + update) of `wl`
    until `budget_s` of CPU work (bounded sample). Returns (samples/s, sample description)."""
    from oracle import emb_oracle as O
    cfg = O.config_from_workload(wl)
    ora = O.OracleEmbedding(cfg)
    B = batch or wl.batch
    done, samples, t_tot, nnz = 0, 0, 0.0, 0
    k = 0
    # a few distinct batches generated up front and cycled (generating one per step cost more wall
    # time than the oracle step itself at small batches and long --steps)
    nb = 4 if max_steps is None else max(1, min(4, max_steps))
    batches = [synthgen.make_batch(wl, rank=0, step=1000 + i, batch=B) for i in range(nb)]
    while t_tot < budget_s and (max_steps is None or done < max_steps):
        bt = batches[k % nb]
        t0 = time.perf_counter()
        ora.lookup([(bt.ids, bt.offsets, bt.batch)])
        ora.backward_update([bt.dy], wl.lr)
        t_tot += time.perf_counter() - t0
        done += 1
        samples += B
        nnz += bt.nnz
        k += 1
    return samples / t_tot, nnz / t_tot, f"{done} oracle step(s) of {wl.name} at batch {B} ({t_tot:.1f} s CPU)"


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        n = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        n = 1
    # the oracle's hot NumPy primitives (unique/sort/add.at/fancy indexing) are single-threaded
    return 1, n


# ------------------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--workload", default=None, help="override (C1..C5) for experiments")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3-at-1-GPU weak-scaling record (N = 1)")
    ap.add_argument("--profile-steps", type=int, default=24,
                    help="untimed steps with per-kernel events after the headline loop")
    ap.add_argument("--opt", default=None, choices=["sgd", "adagrad", "rowwise_adagrad"],
                    help="override the optimizer (experiments; BJ:8 is element-wise Adagrad)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    n = world
    wl = workload_for(n)
    if args.workload:
        wl = synthgen.WORKLOADS[args.workload]
    if args.batch:
        wl = wl.with_(batch=args.batch)
    if args.opt:
        wl = wl.with_(opt=args.opt)

    if args.impl == "reference":
        if rank != 0:
            return
        per_step = 1.3e-4 * 26 / wl.num_slots  # ~s per sample of the oracle (GPU-box host, C2: ~8 k samples/s)
        B = int(max(64, min(wl.batch, 150.0 / max(1, args.steps + args.warmup) / per_step)))
        sps, lps, sample = oracle_time(wl, budget_s=1e9, max_steps=args.steps + args.warmup, batch=B)
        thr, pool = cpu_threads()
        line = {"impl": "reference", "metric": METRIC, "value": sps, "unit": "samples/s", "n_gpus": n,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * B / sps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": describe(wl, n), "batch_per_step": B},
                "lookups_per_s": lps,
                "cpu_baseline": {"value": sps, "unit": "samples/s", "cores": thr, "kind": "oracle",
                                 "sample": sample + f"; host has {os.cpu_count()} cores"},
                "e2e": {"value": sps, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    if n > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_2112_02752_b200 import emb as E

    nccl_id = None
    if n > 1:
        obj = [E.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    def barrier():
        if n > 1:
            dist.barrier()
        torch.cuda.synchronize()

    res = run_workload(wl, args, n, rank, local_rank, nccl_id, barrier, e2e_steps=args.e2e_steps,
                       profile_steps=args.profile_steps)
    # weak-scaling denominator (N = 1 only): C3 -- the workload the N > 1 lines run -- on this one GPU
    c3_w1 = None
    if n == 1 and not args.workload and not args.no_c3:
        r3 = run_workload(synthgen.WORKLOADS["C3"], args, 1, 0, local_rank, None, barrier, e2e_steps=0,
                          profile_steps=0)
        c3_w1 = {"workload": describe(synthgen.WORKLOADS["C3"], 1), "value": r3["value"], "unit": "samples/s",
                 "ms_per_step": r3["ms_per_step"], "step_roofline": r3["step_roofline"],
                 "note": "same config as the N>1 lines (C3, B=16,384 per GPU): the weak-scaling denominator"}

    cpu = None
    if rank == 0 and n == 1 and not args.no_cpu:  # the CPU baseline is an N = 1 figure
        sps, lps, sample = oracle_time(wl, budget_s=args.cpu_budget)
        thr, pool = cpu_threads()
        cpu = {"value": sps, "unit": "samples/s", "cores": thr, "kind": "oracle",
               "sample": sample + f"; host has {os.cpu_count()} cores, NumPy primitives single-threaded",
               "lookups_per_s": lps}

    if rank == 0:
        line = {
            "metric": METRIC, "value": res["value"], "unit": "samples/s", "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 (fp64 accumulation)", "data": "synthetic",
            "config": res["config"],
            "lookups_per_s": res["lookups_per_s"],
            "fwd_ms": res["fwd_ms"],
            "step_roofline": res["step_roofline"],
            "roofline": res["roofline"],
            "nvlink": res["nvlink"],
            "kernels": res["kernels"],
            "cpu_baseline": cpu,
            "e2e": res["e2e"],
            "c3_w1": c3_w1,
            "gpu_launches": res["gpu_launches"],
            "clocks": res["clocks"],
        }
        print(json.dumps(line), flush=True)
    if n > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_workload(wl, args, n, rank, local_rank, nccl_id, barrier, e2e_steps, profile_steps):
    """Time `args.steps` fwd+bwd+update steps of `wl` (inputs resident in HBM) on this rank; returns the
    fields of the JSON line. The headline loop carries no per-kernel events; a separate profiled loop of
    `profile_steps` steps (libemb's event profiler, every kernel on the stream it runs on) gives the
    per-kernel breakdown, the forward time and the dominant kernel's roofline."""
    import torch
    import torch.distributed as dist
    from paper_2112_02752_b200.harness import DeviceBatch, make_layer

    # stage a pool of distinct batches in HBM (inputs resident before the timed region); C4's batches
    # are ~1.8 GB each, so fewer of them (still far above the 126 MB L2)
    nstage = POOL_BATCHES if wl.batch * wl.num_slots * wl.dim * 8 < 500e6 else 4
    host_batches = [synthgen.make_batch(wl, rank=rank, step=i) for i in range(nstage)]
    max_nnz = max(b.nnz for b in host_batches)
    dev_batches = [DeviceBatch(b, wl.num_slots, wl.dim, local_rank) for b in host_batches]
    layer = make_layer(wl, max_batch=wl.batch, max_ids=max_nnz, world=n, rank=rank, nccl_id=nccl_id,
                       device=local_rank)
    stream = torch.cuda.current_stream()
    # emb_lookup_prefetch: the next step's first phase (W = 1: the dedup sort; W > 1: sort + route)
    # declared before this step's backward, which launches it right after its gradient kernel, so it
    # overlaps the gradient passes (a training loop knows its next batch). Default: on, except at
    # N = 2, where the sort's SM time costs the two short gradient passes more than it hides (C3:
    # 281.7 us/step without, 289.8 with; W = 4: 372.3 without, 361.2 with; C2: 137.0 without, 124-125
    # with -- profiles/r02_bench_*prefetch*). EMB_BENCH_PREFETCH=0/1 overrides. Within each loop the
    # first step runs its own first phase and the last prefetches nothing, so every step's work is
    # inside the loop that times it.
    pf_env = os.environ.get("EMB_BENCH_PREFETCH")
    use_prefetch = (pf_env == "1") if pf_env is not None else n != 2

    def step(i, last=False):
        db = dev_batches[i % nstage]
        layer.lookup(db.ids, db.offsets, db.batch, db.nnz, db.out, stream)
        if use_prefetch and not last:
            nx = dev_batches[(i + 1) % nstage]
            layer.lookup_prefetch(nx.ids, nx.offsets, nx.batch, nx.nnz, stream)
        layer.backward_update(db.dy, wl.lr, stream)

    def max_ranks(x):
        if n == 1:
            return x
        t = torch.tensor([x], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for i in range(args.warmup):
        step(i, i == args.warmup - 1)
    barrier()
    # per-step statistics (unique counts) for the byte accounting, outside the timed region
    infos = []
    lo_fracs = []
    for i in range(nstage):
        step(i, i == nstage - 1)
        infos.append(layer.step_info())  # launches counted over lookup + backward
        if n > 1 and i < 2:  # share of received keys with more than one source (they carry the lo half)
            _, fanin = layer.last_owner_unique()
            lo_fracs.append(float(fanin[fanin > 1].sum()) / max(1, int(fanin.sum())))
    barrier()
    layer.profile(True)  # allocates the profiler's event pool now, outside the timed region
    layer.profile(False)
    layer.profile_reset()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            step(i, i == args.steps - 1)
        ev1.record(stream)
        torch.cuda.synchronize()
    t_ms = max_ranks(ev0.elapsed_time(ev1))
    barrier()

    # profiled loop (not part of the headline): per-kernel device times and the forward time
    prof, fwd_ms = {}, float("nan")
    if profile_steps > 0:
        fwd_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(profile_steps)]
        layer.profile(True)
        # no prefetch here: fwd_ms is the whole lookup (sort included) and every kernel's time is its
        # own, not stretched by a concurrent prefetched sort
        for i in range(profile_steps):
            db = dev_batches[i % nstage]
            fwd_ev[i][0].record(stream)
            layer.lookup(db.ids, db.offsets, db.batch, db.nnz, db.out, stream)
            fwd_ev[i][1].record(stream)
            if os.environ.get("EMB_BENCH_PROFILE_PREFETCH") == "1" and use_prefetch and i < profile_steps - 1:
                nx = dev_batches[(i + 1) % nstage]  # (diagnostics: the timed loop's overlap, profiled)
                layer.lookup_prefetch(nx.ids, nx.offsets, nx.batch, nx.nnz, stream)
            layer.backward_update(db.dy, wl.lr, stream)
        torch.cuda.synchronize()
        prof = layer.profile_read()
        layer.profile(False)
        fwd_ms = max_ranks(statistics.mean(a.elapsed_time(b) for a, b in fwd_ev))
        barrier()

    ms_step = t_ms / args.steps
    B = wl.batch
    samples_s = n * B * args.steps / (t_ms / 1e3)
    mean = lambda key: statistics.mean(inf[key] for inf in infos)  # noqa: E731
    N_mean = statistics.mean(b.nnz for b in host_batches)
    SB = wl.num_slots * B
    U_l, U_o = mean("unique_local"), mean("unique_owner")
    lookups_s = n * N_mean / (fwd_ms / 1e3) if fwd_ms == fwd_ms else None
    peak, peak_src = _peaks()
    hbm = step_bytes(wl, N_mean, SB, U_l, U_o, n)
    launches_per_step = statistics.mean(inf["launches"] for inf in infos)

    # dominant kernel = largest summed device time among the step kernels with a byte model (the owner
    # merge / flag kernels run on a side stream, hidden behind the gather-push and the pool)
    modeled = {k: v for k, v in prof.items() if kernel_bytes(k, wl, 1, 1, 1, n, 1) is not None}
    dom, (dom_ms, dom_cnt) = max(modeled.items(), key=lambda kv: kv[1][0]) if modeled else ("none", (0.0, 0))
    kb = kernel_bytes(dom, wl, N_mean, SB, U_o, n, U_l)
    roof = None
    if kb is not None and dom_cnt:
        t_launch = dom_ms / dom_cnt / 1e3
        ach = kb / t_launch / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": _traffic(dom, wl.opt) if n == 1 else None,
                "launch_us": round(t_launch * 1e6, 2), "algorithmic_bytes_per_launch": int(kb),
                "peak_source": peak_src,
                "timing": f"CUDA events on the kernel's stream, {profile_steps} profiled steps after the timed loop"}
    kernels = {k: {"ms_total": round(v[0], 3), "launches": v[1], "us_per_launch": round(1e3 * v[0] / max(v[1], 1), 2)}
               for k, v in prof.items()}
    nvl = None
    if n > 1:
        lo_frac = max_ranks(statistics.mean(lo_fracs)) if lo_fracs else 1.0
        nb = nvlink_bytes(wl, U_l, n, lo_frac)
        ex_us = sum(kernels[k]["us_per_launch"] for k in ("gather_push", "grad_push") if k in kernels)
        nvl = {"bytes_per_step_per_direction": int(nb), "lo_half_share": round(lo_frac, 4), "peak_gbs": 770.0,
               "peak_source": "measured peer copy per direction, B200_PROFILING.md (900 nominal)",
               "achieved_step_gbs": round(nb / (ms_step / 1e3) / 1e9, 1),
               "frac_step": round(nb / (ms_step / 1e3) / 1e9 / 770.0, 4),
               "exchange_kernels_us": round(ex_us, 2),
               "frac_exchange_kernels": round(nb / (ex_us / 1e6) / 1e9 / 770.0, 4) if ex_us else None,
               "note": "frac_exchange_kernels: NVLink bytes / (owner gather-push + requester-merge kernel "
                       "times): the exchange phase's fraction of the link (those kernels also do HBM work)"}

    # e2e through the host-buffer C-ABI entry points (pinned host memory, copies inside the timed region)
    e2e = None
    if e2e_steps > 0:
        hb = host_batches[0]
        ids_h = torch.from_numpy(hb.ids).pin_memory()
        off_h = torch.from_numpy(hb.offsets).pin_memory()
        dy_h = torch.from_numpy(hb.dy).pin_memory()
        out_h = torch.empty((B, wl.num_slots, wl.dim), dtype=torch.float32).pin_memory()
        for _ in range(2):
            layer.lookup_host(ids_h.numpy(), off_h.numpy(), B, hb.nnz, out_h.numpy(), stream)
            layer.backward_update_host(dy_h.numpy(), wl.lr, stream)
        layer.host_sync()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            layer.lookup_host(ids_h.numpy(), off_h.numpy(), B, hb.nnz, out_h.numpy(), stream)
            layer.backward_update_host(dy_h.numpy(), wl.lr, stream)
        layer.host_sync()
        e1.record(stream)
        torch.cuda.synchronize()
        te = max_ranks(e0.elapsed_time(e1))
        e2e = {"value": n * B * e2e_steps / (te / 1e3), "unit": "samples/s",
               "h2d_bytes_per_step": int(hb.ids.nbytes + hb.offsets.nbytes + hb.dy.nbytes),
               "d2h_bytes_per_step": int(out_h.numel() * 4), "ms_per_step": te / e2e_steps,
               "path": "emb_lookup_host + emb_backward_update_host (pinned host buffers; H2D and D2H on the "
                       "library's copy streams, double-buffered), emb_host_sync before the end event"}
    config = {"workload": describe(wl, n), "global_batch": n * B, "nnz_per_gpu": N_mean,
              "unique_local": U_l, "unique_owner": U_o,
              "l2": f"inputs larger than L2: {nstage} distinct staged batches cycled "
                    f"({nstage} x {(hb_bytes(host_batches[0], wl)) / 1e6:.0f} MB) + "
                    f"{layer.rows_local * 4 * (wl.dim + layer.accum_width * (wl.opt != 'sgd')) / 1e9:.1f} GB table "
                    "state per GPU",
              "prefetch": ("emb_lookup_prefetch: the next step's sort + route (W = 1: sort) overlaps each backward "
                           "inside the timed loop" if use_prefetch else "off")}
    out = {"value": samples_s, "ms_per_step": ms_step, "config": config, "lookups_per_s": lookups_s,
           "fwd_ms": fwd_ms,
           "step_roofline": {"bound": "hbm", "algorithmic_bytes": int(hbm),
                             "achieved": round(hbm / (ms_step / 1e3) / 1e9, 1), "peak": peak, "unit": "GB/s",
                             "frac": round(hbm / (ms_step / 1e3) / 1e9 / peak, 4)},
           "roofline": roof, "nvlink": nvl, "kernels": kernels, "e2e": e2e,
           "gpu_launches": int(round(launches_per_step * args.steps)), "clocks": clk.summary()}
    layer.close()
    del dev_batches
    torch.cuda.empty_cache()
    return out


def hb_bytes(bt, wl):
    return bt.ids.nbytes + bt.offsets.nbytes + bt.dy.nbytes + bt.batch * wl.num_slots * wl.dim * 4


if __name__ == "__main__":
    main()
