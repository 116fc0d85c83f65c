"""Thin ctypes binding of libemb.so (include/emb.h). Argument marshalling only: every step of the
embedding path runs in the library's CUDA kernels. There is NO CPU fallback: if libemb.so is
missing this module raises on import of the library.

Pointers: anything with .data_ptr() (torch tensors), a NumPy array (.ctypes.data, host only) or a
plain int. Streams: a torch.cuda.Stream, an int handle, or None (= torch's current stream on the
handle's device, else the legacy default stream).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence, Tuple

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libemb.so")

EMB_OK, EMB_ERR_INVALID, EMB_ERR_RANGE, EMB_ERR_STATE, EMB_ERR_NOMEM, EMB_ERR_CUDA, EMB_ERR_NCCL = range(7)
STATUS_NAMES = ["EMB_OK", "EMB_ERR_INVALID", "EMB_ERR_RANGE", "EMB_ERR_STATE", "EMB_ERR_NOMEM", "EMB_ERR_CUDA",
                "EMB_ERR_NCCL"]
EMB_MAX_WORLD = 16
POOL = {"sum": 0, "mean": 1}
OPT = {"sgd": 0, "adagrad": 1, "rowwise_adagrad": 2}
SHARD = {"cyclic": 0, "block": 1}

# every symbol include/emb.h declares (checked by tests/test_abi.py)
EXPORTED = [
    "emb_create", "emb_create_group", "emb_destroy", "emb_get_unique_id", "emb_lookup", "emb_lookup_prefetch",
    "emb_backward_update", "emb_lookup_group", "emb_backward_update_group", "emb_lookup_prefetch_group",
    "emb_lookup_host", "emb_host_sync",
    "emb_backward_update_host", "emb_read_rows", "emb_write_rows", "emb_last_step_info", "emb_last_unique",
    "emb_last_owner_unique", "emb_rows_local", "emb_profile_enable", "emb_profile_reset", "emb_profile_read",
    "emb_profile_name", "emb_clear_error", "emb_last_error",
]


class EmbError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 7 else status}: {msg}")
        self.status = status


class EmbConfigC(ctypes.Structure):
    _fields_ = [
        ("num_tables", ctypes.c_int32), ("rows", ctypes.POINTER(ctypes.c_int64)),
        ("dim", ctypes.c_int32),
        ("num_slots", ctypes.c_int32), ("slot_table", ctypes.POINTER(ctypes.c_int32)),
        ("pool", ctypes.c_int32), ("opt", ctypes.c_int32),
        ("eps", ctypes.c_double), ("init_accum", ctypes.c_float),
        ("init_seed", ctypes.c_uint64),
        ("max_batch", ctypes.c_int32), ("max_ids", ctypes.c_int64),
        ("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("nccl_id", ctypes.c_void_p),
        ("device", ctypes.c_int32), ("shard", ctypes.c_int32),
    ]


class StepInfoC(ctypes.Structure):
    _fields_ = [
        ("nnz", ctypes.c_int64), ("num_bags", ctypes.c_int64), ("unique_local", ctypes.c_int64),
        ("unique_owner", ctypes.c_int64), ("recv_keys", ctypes.c_int64),
        ("world", ctypes.c_int32), ("launches", ctypes.c_int32),
        ("send_counts", ctypes.c_int64 * EMB_MAX_WORLD), ("recv_counts", ctypes.c_int64 * EMB_MAX_WORLD),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libemb.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2112_02752_b200.build` "
                           "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, u64p, i64p = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p
    L.emb_create.argtypes = [ctypes.POINTER(EmbConfigC), ctypes.POINTER(vp)]
    L.emb_create_group.argtypes = [ctypes.POINTER(EmbConfigC), i32, ctypes.POINTER(vp)]
    L.emb_lookup_group.argtypes = [ctypes.POINTER(vp), i32, ctypes.POINTER(vp), ctypes.POINTER(vp),
                                   ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(vp),
                                   ctypes.POINTER(vp)]
    L.emb_backward_update_group.argtypes = [ctypes.POINTER(vp), i32, ctypes.POINTER(vp), ctypes.c_double,
                                            ctypes.POINTER(vp)]
    L.emb_lookup_prefetch_group.argtypes = [ctypes.POINTER(vp), i32, ctypes.POINTER(vp), ctypes.POINTER(vp),
                                            ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64),
                                            ctypes.POINTER(vp)]
    L.emb_destroy.argtypes = [vp]
    L.emb_get_unique_id.argtypes = [vp]
    L.emb_lookup.argtypes = [vp, vp, vp, i32, i64, vp, vp]
    L.emb_lookup_prefetch.argtypes = [vp, vp, vp, i32, i64, vp]
    L.emb_backward_update.argtypes = [vp, vp, ctypes.c_double, vp]
    L.emb_lookup_host.argtypes = [vp, vp, vp, i32, i64, vp, vp]
    L.emb_backward_update_host.argtypes = [vp, vp, ctypes.c_double, vp]
    L.emb_host_sync.argtypes = [vp]
    L.emb_read_rows.argtypes = [vp, i32, vp, i64, vp, vp]
    L.emb_write_rows.argtypes = [vp, i32, vp, i64, vp, vp]
    L.emb_last_step_info.argtypes = [vp, ctypes.POINTER(StepInfoC)]
    L.emb_last_unique.argtypes = [vp, u64p, i64p, i64, ctypes.POINTER(ctypes.c_int64)]
    L.emb_last_owner_unique.argtypes = [vp, u64p, i64p, i64, ctypes.POINTER(ctypes.c_int64)]
    L.emb_rows_local.argtypes = [vp]
    L.emb_rows_local.restype = ctypes.c_int64
    L.emb_profile_enable.argtypes = [vp, i32]
    L.emb_profile_reset.argtypes = [vp]
    L.emb_profile_read.argtypes = [vp, vp, vp, i32, ctypes.POINTER(ctypes.c_int32)]
    L.emb_profile_name.argtypes = [i32]
    L.emb_profile_name.restype = ctypes.c_char_p
    L.emb_clear_error.argtypes = [vp]
    L.emb_last_error.argtypes = [vp]
    L.emb_last_error.restype = ctypes.c_char_p
    for name in EXPORTED:  # every other entry point returns emb_status_t
        if name not in ("emb_rows_local", "emb_profile_name", "emb_last_error"):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def _ptr(x) -> int:
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    if isinstance(x, np.ndarray):
        return int(x.ctypes.data)
    raise TypeError(f"cannot take a pointer of {type(x)}")


def _stream(s, device: int) -> int:
    if s is None:
        try:
            import torch
            if torch.cuda.is_available():
                return int(torch.cuda.current_stream(device).cuda_stream)
        except Exception:
            pass
        return 0
    if isinstance(s, int):
        return s
    return int(s.cuda_stream)


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = lib().emb_get_unique_id(buf)
    if st != EMB_OK:
        raise EmbError(st, "emb_get_unique_id")
    return buf.raw


def _config(rows, dim, slot_table, pool, opt, eps, init_accum, seed, max_batch, max_ids, rank, world, nid, device,
            shard):
    return EmbConfigC(
        num_tables=len(rows), rows=rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        dim=dim, num_slots=len(slot_table),
        slot_table=slot_table.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
        pool=POOL[pool], opt=OPT[opt], eps=eps, init_accum=init_accum, init_seed=seed,
        max_batch=max_batch, max_ids=max_ids, rank=rank, world=world,
        nccl_id=ctypes.cast(nid, ctypes.c_void_p) if nid is not None else None,
        device=device, shard=SHARD[shard])


class EmbeddingLayer:
    """One rank's handle of the sparse embedding layer (include/emb.h emb_create)."""

    def __init__(self, rows: Sequence[int], dim: int, slot_table: Sequence[int], *, pool: str = "sum",
                 opt: str = "adagrad", eps: float = 1e-6, init_accum: float = 0.0, seed: int = 2112,
                 max_batch: int, max_ids: int, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 device: int = 0, shard: str = "cyclic", _handle=None):
        L = lib()
        self._rows = np.ascontiguousarray(rows, dtype=np.int64)
        self._slots = np.ascontiguousarray(slot_table, dtype=np.int32)
        self._nid = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        if _handle is None:
            cfg = _config(self._rows, dim, self._slots, pool, opt, eps, init_accum, seed, max_batch, max_ids, rank,
                          world, self._nid, device, shard)
            h = ctypes.c_void_p()
            st = L.emb_create(ctypes.byref(cfg), ctypes.byref(h))
            if st != EMB_OK:
                raise EmbError(st, L.emb_last_error(None).decode())
            self.h = h
        else:
            self.h = _handle
        self.dim, self.num_slots, self.device, self.world, self.rank = dim, len(self._slots), device, world, rank
        self.rows = tuple(int(r) for r in self._rows)
        self.slot_table = tuple(int(s) for s in self._slots)
        self.pool, self.opt = pool, opt

    # ---- helpers
    def _check(self, st: int, what: str):
        if st != EMB_OK:
            raise EmbError(st, f"{what}: {lib().emb_last_error(self.h).decode()}")

    def close(self):
        if getattr(self, "h", None):
            lib().emb_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def rows_local(self) -> int:
        return int(lib().emb_rows_local(self.h))

    # ---- the step
    def lookup(self, ids, offsets, batch: int, nnz: int, out, stream=None):
        self._check(lib().emb_lookup(self.h, _ptr(ids), _ptr(offsets), int(batch), int(nnz), _ptr(out),
                                     _stream(stream, self.device)), "emb_lookup")

    def lookup_prefetch(self, ids, offsets, batch: int, nnz: int, stream=None):
        """Declare the NEXT lookup's inputs: the next backward launches their dedup sort (W > 1: sort +
        route) right after its gradient kernel, overlapping it (include/emb.h emb_lookup_prefetch)."""
        self._check(lib().emb_lookup_prefetch(self.h, _ptr(ids), _ptr(offsets), int(batch), int(nnz),
                                              _stream(stream, self.device)), "emb_lookup_prefetch")

    def backward_update(self, d_out, lr: float, stream=None):
        self._check(lib().emb_backward_update(self.h, _ptr(d_out), float(lr), _stream(stream, self.device)),
                    "emb_backward_update")

    def lookup_host(self, ids: np.ndarray, offsets: np.ndarray, batch: int, nnz: int, out: np.ndarray, stream=None):
        self._check(lib().emb_lookup_host(self.h, _ptr(ids), _ptr(offsets), int(batch), int(nnz), _ptr(out),
                                          _stream(stream, self.device)), "emb_lookup_host")

    def backward_update_host(self, d_out: np.ndarray, lr: float, stream=None):
        self._check(lib().emb_backward_update_host(self.h, _ptr(d_out), float(lr), _stream(stream, self.device)),
                    "emb_backward_update_host")

    def host_sync(self):
        """Wait for every host-buffer call (asynchronous: the buffers must stay untouched until then)."""
        self._check(lib().emb_host_sync(self.h), "emb_host_sync")

    # ---- host-synchronous helpers
    def read_rows(self, table: int, rows) -> Tuple[np.ndarray, np.ndarray]:
        r = np.ascontiguousarray(rows, dtype=np.int64)
        w = np.empty((r.size, self.dim), np.float32)
        a = np.empty((r.size, self.accum_width), np.float32)
        self._check(lib().emb_read_rows(self.h, table, _ptr(r), r.size, _ptr(w), _ptr(a)), "emb_read_rows")
        return w, a

    @property
    def accum_width(self) -> int:
        """Optimizer-state floats per row: 1 for row-wise Adagrad, else D."""
        return 1 if self.opt == "rowwise_adagrad" else self.dim

    def write_rows(self, table: int, rows, w, a=None):
        r = np.ascontiguousarray(rows, dtype=np.int64)
        w = np.ascontiguousarray(w, dtype=np.float32)
        a = None if a is None else np.ascontiguousarray(a, dtype=np.float32)
        self._check(lib().emb_write_rows(self.h, table, _ptr(r), r.size, _ptr(w), _ptr(a)), "emb_write_rows")

    def step_info(self) -> dict:
        info = StepInfoC()
        self._check(lib().emb_last_step_info(self.h, ctypes.byref(info)), "emb_last_step_info")
        W = info.world
        return dict(nnz=info.nnz, num_bags=info.num_bags, unique_local=info.unique_local,
                    unique_owner=info.unique_owner, recv_keys=info.recv_keys, world=W, launches=info.launches,
                    send_counts=list(info.send_counts)[:W], recv_counts=list(info.recv_counts)[:W])

    def _unique(self, fn):
        n = ctypes.c_int64()
        fn(self.h, None, None, 0, ctypes.byref(n))  # query the size (returns EMB_ERR_INVALID if cap < n)
        keys = np.empty(max(n.value, 1), np.uint64)
        cnts = np.empty(max(n.value, 1), np.int64)
        self._check(fn(self.h, _ptr(keys), _ptr(cnts), keys.size, ctypes.byref(n)), "unique")
        return keys[:n.value], cnts[:n.value]

    def last_unique(self):
        """GPU dedup of the last batch: sorted distinct fused keys g and their multiplicities."""
        return self._unique(lib().emb_last_unique)

    def last_owner_unique(self):
        """Owner side: sorted distinct owned fused keys requested in the last step, and their fan-in."""
        return self._unique(lib().emb_last_owner_unique)

    def profile(self, on: bool = True):
        self._check(lib().emb_profile_enable(self.h, int(on)), "emb_profile_enable")

    def profile_reset(self):
        self._check(lib().emb_profile_reset(self.h), "emb_profile_reset")

    def profile_read(self) -> dict:
        ms = (ctypes.c_double * 32)()
        cnt = (ctypes.c_int64 * 32)()
        n = ctypes.c_int32()
        self._check(lib().emb_profile_read(self.h, ms, cnt, 32, ctypes.byref(n)), "emb_profile_read")
        return {lib().emb_profile_name(k).decode(): (ms[k], cnt[k]) for k in range(n.value) if cnt[k] > 0}

    def clear_error(self):
        self._check(lib().emb_clear_error(self.h), "emb_clear_error")

    def last_error(self) -> str:
        return lib().emb_last_error(self.h).decode()


class EmbeddingGroup:
    """All `world` ranks of a row-sharded layer in this process (include/emb.h emb_create_group): rank r
    on devices[r] (devices may repeat: several ranks emulated on one GPU). Step with lookup() /
    backward_update() over per-rank argument lists; .layers[r] gives the per-rank helpers (read_rows,
    step_info, last_unique, ...)."""

    def __init__(self, rows: Sequence[int], dim: int, slot_table: Sequence[int], *, world: int,
                 devices: Optional[Sequence[int]] = None, pool: str = "sum", opt: str = "adagrad", eps: float = 1e-6,
                 init_accum: float = 0.0, seed: int = 2112, max_batch: int, max_ids, shard: str = "cyclic"):
        L = lib()
        devices = list(devices) if devices is not None else [0] * world
        max_ids = list(max_ids) if isinstance(max_ids, (list, tuple)) else [int(max_ids)] * world
        self._rows = np.ascontiguousarray(rows, dtype=np.int64)
        self._slots = np.ascontiguousarray(slot_table, dtype=np.int32)
        cfgs = (EmbConfigC * world)(*[
            _config(self._rows, dim, self._slots, pool, opt, eps, init_accum, seed, max_batch, max_ids[r], r, world,
                    None, devices[r], shard) for r in range(world)])
        hs = (ctypes.c_void_p * world)()
        st = L.emb_create_group(cfgs, world, hs)
        if st != EMB_OK:
            raise EmbError(st, L.emb_last_error(None).decode())
        self._hs = hs
        self.world, self.devices = world, devices
        self.layers = [EmbeddingLayer(rows, dim, slot_table, pool=pool, opt=opt, eps=eps, init_accum=init_accum,
                                      seed=seed, max_batch=max_batch, max_ids=max_ids[r], rank=r, world=world,
                                      device=devices[r], shard=shard, _handle=ctypes.c_void_p(hs[r]))
                       for r in range(world)]

    def _streams(self, streams):
        if streams is None:
            streams = [None] * self.world
        return (ctypes.c_void_p * self.world)(*[_stream(s, d) for s, d in zip(streams, self.devices)])

    def lookup(self, ids, offsets, batch, nnz, out, streams=None):
        W = self.world
        st = lib().emb_lookup_group(self._hs, W, (ctypes.c_void_p * W)(*[_ptr(x) for x in ids]),
                                    (ctypes.c_void_p * W)(*[_ptr(x) for x in offsets]),
                                    (ctypes.c_int32 * W)(*[int(b) for b in batch]),
                                    (ctypes.c_int64 * W)(*[int(n) for n in nnz]),
                                    (ctypes.c_void_p * W)(*[_ptr(x) for x in out]), self._streams(streams))
        if st != EMB_OK:
            raise EmbError(st, "emb_lookup_group: " + "; ".join(l.last_error() for l in self.layers))

    def lookup_prefetch(self, ids, offsets, batch, nnz, streams=None):
        W = self.world
        st = lib().emb_lookup_prefetch_group(self._hs, W, (ctypes.c_void_p * W)(*[_ptr(x) for x in ids]),
                                             (ctypes.c_void_p * W)(*[_ptr(x) for x in offsets]),
                                             (ctypes.c_int32 * W)(*[int(b) for b in batch]),
                                             (ctypes.c_int64 * W)(*[int(n) for n in nnz]), self._streams(streams))
        if st != EMB_OK:
            raise EmbError(st, "emb_lookup_prefetch_group: " + "; ".join(l.last_error() for l in self.layers))

    def backward_update(self, d_out, lr: float, streams=None):
        W = self.world
        st = lib().emb_backward_update_group(self._hs, W, (ctypes.c_void_p * W)(*[_ptr(x) for x in d_out]),
                                             float(lr), self._streams(streams))
        if st != EMB_OK:
            raise EmbError(st, "emb_backward_update_group: " + "; ".join(l.last_error() for l in self.layers))

    def close(self):
        for l in getattr(self, "layers", []):
            l.close()
        self.layers = []
