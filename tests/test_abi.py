"""CPU checks of the C-ABI boundary (-m "not gpu"): libemb.so builds, loads, exports every symbol
include/emb.h declares, the ctypes structs match the header's layout, and argument validation that
happens before any device call returns the documented status codes."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "emb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(emb_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2112_02752_b200 import build
    build.build()
    from paper_2112_02752_b200 import emb
    return emb.lib()


def test_exports_every_declared_symbol(L):
    from paper_2112_02752_b200 import emb
    declared = _declared_symbols()
    assert declared, "no declarations parsed"
    assert sorted(emb.EXPORTED) == declared
    for name in declared:
        assert hasattr(L, name), name


def test_struct_layout_matches_header(L):
    from paper_2112_02752_b200 import emb
    # emb_config_t: offsets implied by the C struct (x86-64 SysV)
    f = dict((n, getattr(emb.EmbConfigC, n).offset) for n, _ in emb.EmbConfigC._fields_)
    assert f["rows"] == 8 and f["dim"] == 16 and f["slot_table"] == 24 and f["eps"] == 40
    assert f["init_seed"] == 56 and f["max_ids"] == 72 and f["nccl_id"] == 88
    assert ctypes.sizeof(emb.EmbConfigC) == 104
    assert ctypes.sizeof(emb.StepInfoC) == 5 * 8 + 8 + 2 * 16 * 8


def _cfg(emb, **kw):
    rows = np.array(kw.pop("rows", [100]), np.int64)
    slots = np.array(kw.pop("slots", [0]), np.int32)
    c = emb.EmbConfigC(num_tables=len(rows), rows=rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), dim=16,
                       num_slots=len(slots), slot_table=slots.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                       pool=0, opt=1, eps=1e-6, init_accum=0.0, init_seed=1, max_batch=8, max_ids=64, rank=0,
                       world=1, nccl_id=None, device=0, shard=0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c, (rows, slots)


@pytest.mark.parametrize("field,value", [("dim", 6), ("dim", 0), ("dim", 260), ("eps", 0.0), ("max_batch", 0),
                                         ("max_ids", 0), ("world", 0), ("rank", 3), ("pool", 7), ("opt", 9),
                                         ("shard", 5), ("num_tables", 0)])
def test_invalid_config_rejected_before_device(L, field, value):
    from paper_2112_02752_b200 import emb
    c, keep = _cfg(emb, **{field: value})
    h = ctypes.c_void_p()
    st = L.emb_create(ctypes.byref(c), ctypes.byref(h))
    assert st == emb.EMB_ERR_INVALID and not h.value
    assert L.emb_last_error(None)


def test_world_without_nccl_id_rejected(L):
    from paper_2112_02752_b200 import emb
    c, keep = _cfg(emb, world=2)
    h = ctypes.c_void_p()
    assert L.emb_create(ctypes.byref(c), ctypes.byref(h)) == emb.EMB_ERR_INVALID


def test_null_handle_calls_are_errors_not_crashes(L):
    from paper_2112_02752_b200 import emb
    assert L.emb_lookup(None, None, None, 0, 0, None, None) == emb.EMB_ERR_INVALID
    assert L.emb_backward_update(None, None, 0.1, None) == emb.EMB_ERR_INVALID
    assert L.emb_destroy(None) == emb.EMB_OK
    assert L.emb_rows_local(None) == -1
    assert L.emb_profile_name(3) == b"pool"


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-GPU error path")
def test_create_without_gpu_fails_cleanly(L):
    from paper_2112_02752_b200 import emb
    c, keep = _cfg(emb)
    h = ctypes.c_void_p()
    st = L.emb_create(ctypes.byref(c), ctypes.byref(h))
    assert st in (emb.EMB_ERR_CUDA, emb.EMB_ERR_NOMEM) and not h.value
