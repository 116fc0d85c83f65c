"""GPU parity of the CUDA path (through the C-ABI) against the CPU oracle, element by element on the
same seeded inputs. Tolerance (BJ:5 / R21): |gpu - oracle| <= 1e-6 + 1e-5*|oracle| for pooled
outputs and updated rows; unique sets, counts and routing bit-exact; run-to-run bitwise determinism.
Multi-step comparisons follow the stepwise-resynced protocol (R22) unless stated free-running."""
import numpy as np
import pytest

import synthgen
from oracle import emb_oracle as O

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-6


@pytest.fixture(scope="module")
def torch():
    t = pytest.importorskip("torch")
    if not t.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2112_02752_b200 import build
    build.build()
    return t


def _layer(wl, B, nnz_cap, **kw):
    from paper_2112_02752_b200.harness import make_layer
    return make_layer(wl, max_batch=B, max_ids=max(nnz_cap, 1), **kw)


def _run_step(torch, layer, bt, lr, dy=None):
    from paper_2112_02752_b200.harness import DeviceBatch
    db = DeviceBatch(bt, layer.num_slots, layer.dim, layer.device)
    layer.lookup(db.ids, db.offsets, db.batch, db.nnz, db.out)
    torch.cuda.synchronize()
    Y = db.out.cpu().numpy()
    info = layer.step_info()
    keys, counts = layer.last_unique()
    d = db.dy if dy is None else torch.from_numpy(dy).cuda()
    layer.backward_update(d, lr)
    torch.cuda.synchronize()
    return Y, info, keys, counts


def _touched_rows(cfg, bt):
    g, _, _ = O.occurrence_keys(cfg, bt.ids, bt.offsets, bt.batch)
    return np.unique(g)


def _read_global(layer, cfg, g):
    """Read fused rows g (all owned by this W=1 layer) -> (w, a)."""
    t = np.searchsorted(cfg.base, g, side="right") - 1
    w = np.empty((g.size, cfg.dim), np.float32)
    a = np.empty((g.size, cfg.accum_width), np.float32)
    for tt in np.unique(t):
        m = t == tt
        w[m], a[m] = layer.read_rows(int(tt), g[m] - cfg.base[tt])
    return w, a


def _check_close(gpu, ref, what):
    err = np.abs(gpu.astype(np.float64) - ref.astype(np.float64))
    bound = ATOL + RTOL * np.abs(ref.astype(np.float64))
    bad = err > bound
    assert not bad.any(), f"{what}: {bad.sum()} elements out of tolerance, worst {np.max(err / bound):.3g}x"


def _parity_run(torch, wl, B, steps, lr, resync=True, empty_frac=0.0, check_all_rows=False):
    cfg = O.config_from_workload(wl)
    bts = [synthgen.make_batch(wl, step=k, batch=B, empty_frac=empty_frac) for k in range(steps)]
    layer = _layer(wl, B, max(bt.nnz for bt in bts))
    ora = O.OracleEmbedding(cfg)
    try:
        for k, bt in enumerate(bts):
            touched = _touched_rows(cfg, bt)
            if resync and k > 0:
                w, a = _read_global(layer, cfg, touched)
                ora.load_rows(touched, w, a)
            Y, info, keys, counts = _run_step(torch, layer, bt, lr)
            (Yo,) = ora.lookup([(bt.ids, bt.offsets, bt.batch)])
            _check_close(Y, Yo, f"Y step {k}")
            g, _, _ = O.occurrence_keys(cfg, bt.ids, bt.offsets, bt.batch)
            Uo, co, _ = O.dedup(g)
            assert np.array_equal(keys.astype(np.int64), Uo), "unique set differs"
            assert np.array_equal(counts, co), "counts differ"
            assert info["unique_local"] == Uo.size and info["nnz"] == bt.nnz
            ora.backward_update([bt.dy], lr)
            rows = np.arange(cfg.total_rows) if check_all_rows else touched
            w, a = _read_global(layer, cfg, rows)
            wo, ao = ora.rows(rows)
            _check_close(w, wo, f"w step {k}")
            if wl.opt in ("adagrad", "rowwise_adagrad"):
                _check_close(a, ao, f"a step {k}")
    finally:
        layer.close()


# ----------------------------------------------------------------------------- C1 (BJ:7) and variants
def test_c1_full_config_free_running(torch):
    """C1 exactly as BJ:7 (uniform ids, SGD, sum): free-running 4 steps, whole table compared."""
    wl = synthgen.WORKLOADS["C1"]
    _parity_run(torch, wl, wl.batch, steps=4, lr=wl.lr, resync=False, check_all_rows=True)


@pytest.mark.parametrize("pool", ["sum", "mean"])
@pytest.mark.parametrize("opt", ["sgd", "adagrad"])
def test_c1_pool_opt_matrix(torch, pool, opt):
    wl = synthgen.WORKLOADS["C1"].with_(pool=pool, opt=opt, ids="zipf", zipf_s=1.2)
    _parity_run(torch, wl, 777, steps=3, lr=0.05, empty_frac=0.1)


@pytest.mark.parametrize("dim", [4, 16, 64, 100, 128, 256])
def test_dims(torch, dim):
    wl = synthgen.WORKLOADS["C1"].with_(dim=dim, rows=(5000, 3000), slot_table=(0, 1, 1), ids="zipf", zipf_s=1.1,
                                        opt="adagrad", pool="mean")
    _parity_run(torch, wl, 300, steps=2, lr=0.1, empty_frac=0.05)


# row-wise Adagrad (reading R14'): compile-time dims, the generic-D path (100), mean
# pooling and the long hot segments that cross warp ranges (ticket combine)
@pytest.mark.parametrize("dim,pool", [(16, "sum"), (64, "mean"), (100, "sum"), (128, "sum"), (256, "mean")])
def test_rowwise_adagrad_dims(torch, dim, pool):
    wl = synthgen.WORKLOADS["C1"].with_(dim=dim, rows=(5000, 3000), slot_table=(0, 1, 1), ids="zipf", zipf_s=1.1,
                                        opt="rowwise_adagrad", pool=pool, init_accum=0.1)
    _parity_run(torch, wl, 300, steps=3, lr=0.1, empty_frac=0.05)


def test_rowwise_adagrad_c2_and_hot(torch):
    _parity_run(torch, synthgen.WORKLOADS["C2"].with_(opt="rowwise_adagrad"), 1024, steps=2, lr=0.01)
    _parity_run(torch, synthgen.WORKLOADS["C5"].with_(opt="rowwise_adagrad"), 128, steps=2, lr=0.01)


def test_c2_full_size(torch):
    """C2 at BASELINE's full size (BJ:8: 26 x 10M rows, D=64, B=16,384, Zipf 1.05, Adagrad) through the
    same device-buffer C-ABI calls bench.py times: every output Y and every touched row of two
    resynced steps against the oracle (the oracle handles this size in seconds)."""
    wl = synthgen.WORKLOADS["C2"]
    _parity_run(torch, wl, wl.batch, steps=2, lr=wl.lr)


def test_c4_like_large_keyspace(torch):
    """C4's structure (BJ:10, R19: 26 slots sharing ONE table, Zipf 1.2) on a 3e8-row table (29-bit
    keys: four radix passes in the per-table sort), D=32 and SGD so the shard fits one GPU; the full
    1e9-row x D=128 C4 needs 4-8 GPUs."""
    wl = synthgen.WORKLOADS["C4"].with_(rows=(300_000_000,), dim=32, opt="sgd")
    _parity_run(torch, wl, 2048, steps=2, lr=0.05)


@pytest.mark.parametrize("opt", ["sgd", "adagrad", "rowwise_adagrad"])
def test_general_sort_path(torch, opt):
    """A non-monotone slot -> table map (slot 0 -> table 1, slot 1 -> table 0) cannot use the per-table
    sort: the key kernel + the general LSD radix sort + the key-mode pool run instead."""
    wl = synthgen.WORKLOADS["C1"].with_(rows=(50_000, 30_000), slot_table=(1, 0, 1), ids="zipf", zipf_s=1.1,
                                        opt=opt, pool="mean")
    _parity_run(torch, wl, 700, steps=3, lr=0.05, empty_frac=0.05)


def test_c2_reduced_batch_full_tables(torch):
    """C2 tables (26 x 10M, D=64, Zipf 1.05, Adagrad) with a reduced batch: 3 resynced steps."""
    wl = synthgen.WORKLOADS["C2"]
    _parity_run(torch, wl, 1024, steps=3, lr=wl.lr)


def test_c5_hot_ids_reduced(torch):
    """C5 hot-id stress (bag 64, 90% of ids in the top-1k rows per table) at one rank, B=256:
    long duplicate segments exercise the multi-chunk ticket combine."""
    wl = synthgen.WORKLOADS["C5"]
    _parity_run(torch, wl, 256, steps=2, lr=wl.lr)


# ----------------------------------------------------------------------------- edge cases
def _hand_batch(ids, offsets, B, S, D, seed=0):
    rng = np.random.default_rng(seed)
    return synthgen.Batch(ids=np.asarray(ids, np.int64), offsets=np.asarray(offsets, np.int64), batch=B,
                          dy=(rng.random((B, S, D), dtype=np.float32) * 2 - 1).astype(np.float32))


def _edge_run(torch, wl, bt, lr=0.1, steps=1):
    cfg = O.config_from_workload(wl)
    layer = _layer(wl, max(bt.batch, 1), max(bt.nnz, 1))
    ora = O.OracleEmbedding(cfg)
    try:
        for _ in range(steps):
            Y, info, keys, counts = _run_step(torch, layer, bt, lr)
            (Yo,) = ora.lookup([(bt.ids, bt.offsets, bt.batch)])
            _check_close(Y, Yo, "Y")
            ora.backward_update([bt.dy], lr)
            rows = np.arange(cfg.total_rows)
            w, a = _read_global(layer, cfg, rows)
            _check_close(w, ora.rows(rows)[0], "w")
    finally:
        layer.close()


def test_one_id_repeated_many_times(torch):
    """A single row hit 5000 times (a segment spanning ~157 chunks) plus a few others."""
    wl = synthgen.WORKLOADS["C1"].with_(rows=(64,), slot_table=(0,), dim=16, opt="adagrad")
    ids = np.concatenate([np.full(5000, 7), np.arange(20) % 64, np.full(100, 63)])
    B = 50
    lens = np.full(B, ids.size // B)
    lens[-1] += ids.size - lens.sum()
    offs = np.concatenate([[0], np.cumsum(lens)])
    _edge_run(torch, wl, _hand_batch(ids, offs, B, 1, 16), steps=2)


@pytest.mark.parametrize("opt", ["adagrad", "rowwise_adagrad"])
def test_single_row_tables(torch, opt):
    """Degenerate tables: one with a single row (every id is 0: one segment holding all of its
    occurrences; 1-bit keys, one radix pass) next to a 7-row table, Zipf ids, empty bags."""
    wl = synthgen.WORKLOADS["C1"].with_(rows=(1, 7), slot_table=(0, 1), dim=16, opt=opt, ids="zipf", zipf_s=1.1)
    _parity_run(torch, wl, 300, steps=3, lr=0.05, empty_frac=0.1)


def test_all_empty_bags_and_max_id(torch):
    wl = synthgen.WORKLOADS["C1"].with_(rows=(10, 5), slot_table=(0, 1), dim=8, opt="sgd")
    ids = np.array([9, 4, 4, 0])
    offs = np.array([0, 0, 0, 2, 2, 2, 4])  # S=2, B=3: bags (0,0)=[], (0,1)=[], (0,2)=[9,4], (1,*)=[],[],[4,0]
    _edge_run(torch, wl, _hand_batch(ids, offs, 3, 2, 8))


def test_batch_zero_and_nnz_zero(torch):
    wl = synthgen.WORKLOADS["C1"].with_(rows=(10,), slot_table=(0,), dim=8)
    _edge_run(torch, wl, _hand_batch([], [0, 0, 0, 0], 3, 1, 8))
    layer = _layer(wl, 4, 4)
    try:
        out = torch.empty((0, 1, 8), device="cuda")
        layer.lookup(torch.zeros(1, dtype=torch.int64, device="cuda"),
                     torch.zeros(1, dtype=torch.int64, device="cuda"), 0, 0, out)
        layer.backward_update(out, 0.1)
        torch.cuda.synchronize()
    finally:
        layer.close()


def test_determinism_bitwise(torch):
    wl = synthgen.WORKLOADS["C5"].with_(rows=(200_000,) * 4, slot_table=(0, 1, 2, 3), bag_len=32)
    bts = [synthgen.make_batch(wl, step=k, batch=512) for k in range(2)]
    res = []
    for _ in range(2):
        layer = _layer(wl, 512, bts[0].nnz)
        Ys = [_run_step(torch, layer, bt, 0.01)[0] for bt in bts]
        g = np.arange(0, 200_000, 7)
        w, a = layer.read_rows(1, g)
        res.append((Ys, w, a))
        layer.close()
    for y0, y1 in zip(res[0][0], res[1][0]):
        assert np.array_equal(y0.view(np.uint32), y1.view(np.uint32))
    assert np.array_equal(res[0][1].view(np.uint32), res[1][1].view(np.uint32))
    assert np.array_equal(res[0][2].view(np.uint32), res[1][2].view(np.uint32))


@pytest.mark.parametrize("wname", ["C2", "C5"])
def test_prefetch_matches_plain_bitwise_and_oracle(torch, wname):
    """emb_lookup_prefetch (the next step's sort, declared before this step's backward and launched by
    it, overlapping the gradient pass) gives bitwise the same Y and rows as the plain path, and matches
    the oracle; a prefetch whose inputs differ from the next lookup's is discarded."""
    from paper_2112_02752_b200.harness import DeviceBatch
    wl = synthgen.WORKLOADS[wname]
    B = 2048 if wname == "C2" else 128
    steps = 4
    bts = [synthgen.make_batch(wl, step=k, batch=B) for k in range(steps)]
    cfg = O.config_from_workload(wl)
    touched = np.unique(np.concatenate([_touched_rows(cfg, bt) for bt in bts]))
    res = []
    for mode in ("plain", "prefetch"):
        layer = _layer(wl, B, max(bt.nnz for bt in bts))
        dbs = [DeviceBatch(bt, wl.num_slots, wl.dim, layer.device) for bt in bts]
        decoy = DeviceBatch(synthgen.make_batch(wl, step=99, batch=B), wl.num_slots, wl.dim, layer.device)
        Ys = []
        for k, db in enumerate(dbs):
            layer.lookup(db.ids, db.offsets, db.batch, db.nnz, db.out)
            if mode == "prefetch":
                if k == 1:  # a prefetch for other inputs: the next lookup must discard it
                    layer.lookup_prefetch(decoy.ids, decoy.offsets, decoy.batch, decoy.nnz)
                elif k + 1 < steps:
                    nx = dbs[k + 1]
                    layer.lookup_prefetch(nx.ids, nx.offsets, nx.batch, nx.nnz)
            layer.backward_update(db.dy, wl.lr)
            torch.cuda.synchronize()
            Ys.append(db.out.cpu().numpy())
        res.append((Ys, _read_global(layer, cfg, touched)))
        layer.close()
    for y0, y1 in zip(res[0][0], res[1][0]):
        assert np.array_equal(y0.view(np.uint32), y1.view(np.uint32))
    assert np.array_equal(res[0][1][0].view(np.uint32), res[1][1][0].view(np.uint32))
    assert np.array_equal(res[0][1][1].view(np.uint32), res[1][1][1].view(np.uint32))
    # and the prefetch path against the oracle, free-running (R22 tolerance per step is not needed:
    # compare step 0 exactly and the final rows within R21 after a stepwise oracle run)
    ora = O.OracleEmbedding(cfg)
    (Yo,) = ora.lookup([(bts[0].ids, bts[0].offsets, bts[0].batch)])
    _check_close(res[1][0][0], Yo, "prefetch Y step 0")


def test_first_forward_bit_exact(torch):
    """R15: with the hash init every partial sum is exact in fp32, so step 0's Y is bit-exact."""
    wl = synthgen.WORKLOADS["C2"]
    cfg = O.config_from_workload(wl)
    bt = synthgen.make_batch(wl, batch=2048)
    layer = _layer(wl, 2048, bt.nnz)
    try:
        Y, *_ = _run_step(torch, layer, bt, 0.0)
    finally:
        layer.close()
    (Yo,) = O.OracleEmbedding(cfg).lookup([(bt.ids, bt.offsets, bt.batch)])
    assert np.array_equal(Y.view(np.uint32), Yo.view(np.uint32))


# ----------------------------------------------------------------------------- errors and protocol
def test_out_of_range_id_sticky_and_no_update(torch):
    from paper_2112_02752_b200.emb import EmbError, EMB_ERR_RANGE
    wl = synthgen.WORKLOADS["C1"].with_(rows=(10,), slot_table=(0,), dim=8, opt="sgd")
    layer = _layer(wl, 4, 8)
    try:
        w0, _ = layer.read_rows(0, np.arange(10))
        bt = _hand_batch([1, 10, 3], [0, 2, 3], 2, 1, 8)
        from paper_2112_02752_b200.harness import DeviceBatch
        db = DeviceBatch(bt, 1, 8)
        layer.lookup(db.ids, db.offsets, 2, 3, db.out)
        torch.cuda.synchronize()
        with pytest.raises(EmbError) as ei:
            layer.backward_update(db.dy, 0.1)
        assert ei.value.status == EMB_ERR_RANGE
        # the bad id contributed nothing to the forward: bag 0 = row 1 only
        np.testing.assert_array_equal(db.out.cpu().numpy()[0, 0], w0[1])
        with pytest.raises(EmbError):
            layer.lookup(db.ids, db.offsets, 2, 3, db.out)
        layer.clear_error()
        w1, _ = layer.read_rows(0, np.arange(10))
        assert np.array_equal(w0, w1)
    finally:
        layer.close()


def test_bad_offsets_and_state_errors(torch):
    from paper_2112_02752_b200.emb import EmbError, EMB_ERR_INVALID, EMB_ERR_STATE
    wl = synthgen.WORKLOADS["C1"].with_(rows=(10,), slot_table=(0,), dim=8)
    layer = _layer(wl, 4, 8)
    try:
        from paper_2112_02752_b200.harness import DeviceBatch
        with pytest.raises(EmbError) as ei:
            layer.backward_update(torch.zeros(8, device="cuda"), 0.1)
        assert ei.value.status == EMB_ERR_STATE
        db = DeviceBatch(_hand_batch([1, 2, 3], [0, 2, 1, 3], 3, 1, 8), 1, 8)
        layer.lookup(db.ids, db.offsets, 3, 3, db.out)
        torch.cuda.synchronize()
        with pytest.raises(EmbError) as ei:
            layer.backward_update(db.dy, 0.1)
        assert ei.value.status == EMB_ERR_INVALID
        layer.clear_error()
        with pytest.raises(EmbError) as ei:  # argument error: nnz above capacity
            layer.lookup(db.ids, db.offsets, 3, 9, db.out)
        assert ei.value.status == EMB_ERR_INVALID
        db2 = DeviceBatch(_hand_batch([1, 2, 3], [0, 1, 2, 3], 3, 1, 8), 1, 8)
        layer.lookup(db2.ids, db2.offsets, 3, 3, db2.out)
        with pytest.raises(EmbError) as ei:
            layer.lookup(db2.ids, db2.offsets, 3, 3, db2.out)
        assert ei.value.status == EMB_ERR_STATE
    finally:
        layer.close()


def test_read_write_rows_roundtrip_bitwise(torch):
    wl = synthgen.WORKLOADS["C1"].with_(rows=(1000, 500), slot_table=(0, 1), dim=16, opt="adagrad")
    layer = _layer(wl, 8, 64)
    try:
        rows = np.array([0, 5, 499])
        w = np.random.default_rng(0).random((3, 16), dtype=np.float32)
        a = np.random.default_rng(1).random((3, 16), dtype=np.float32)
        layer.write_rows(1, rows, w, a)
        w2, a2 = layer.read_rows(1, rows)
        assert np.array_equal(w, w2) and np.array_equal(a, a2)
        w0, _ = layer.read_rows(0, rows)
        cfg = O.config_from_workload(wl)
        assert np.array_equal(w0, O.init_weights(cfg.seed, rows, 16))  # hash init bitwise (R15)
    finally:
        layer.close()


def test_host_buffer_path(torch):
    """The asynchronous host-buffer entry points (double-buffered staging, H2D / D2H copy streams): four
    steps enqueued back to back with no synchronisation in between (each step's pinned buffers kept
    alive), then emb_host_sync; every step's Y and the final rows match the free-running oracle."""
    wl = synthgen.WORKLOADS["C1"].with_(ids="zipf", zipf_s=1.2, opt="adagrad")
    cfg = O.config_from_workload(wl)
    bts = [synthgen.make_batch(wl, step=k, batch=256) for k in range(4)]
    layer = _layer(wl, 256, max(bt.nnz for bt in bts))
    ora = O.OracleEmbedding(cfg)
    try:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        ins = [(pin(bt.ids), pin(bt.offsets), pin(bt.dy)) for bt in bts]
        outs = [torch.empty((256, wl.num_slots, wl.dim), dtype=torch.float32).pin_memory() for _ in bts]
        for (i_, o_, d_), out, bt in zip(ins, outs, bts):
            layer.lookup_host(i_.numpy(), o_.numpy(), 256, bt.nnz, out.numpy())
            layer.backward_update_host(d_.numpy(), 0.05)
        layer.host_sync()
        for k, bt in enumerate(bts):
            (Yo,) = ora.lookup([(bt.ids, bt.offsets, 256)])
            ora.backward_update([bt.dy], 0.05)
            _check_close(outs[k].numpy(), Yo, f"Y host path step {k}")
        g = np.unique(np.concatenate([_touched_rows(cfg, bt) for bt in bts]))
        w, a = _read_global(layer, cfg, g)
        _check_close(w, ora.rows(g)[0], "w host path")
        _check_close(a, ora.rows(g)[1], "a host path")
    finally:
        layer.close()


@pytest.mark.parametrize("opt", ["adagrad", "rowwise_adagrad"])
@pytest.mark.parametrize("lr", [1.0, 10.0])
def test_adagrad_large_lr_extreme_values(torch, opt, lr):
    """Reading R16' at its limits: learning rates 1 (fast fp32 sink: sqrt/rcp approximations, error
    <= ~lr*3e-7) and 10 (the fp64 sink, switched on for lr > 1), with huge merged gradients (|G| ~ 1e4),
    subnormal ones (dY ~ 1e-40), accumulators far above 1 (a = 1e6) and near 0, and weights near 0 --
    against the oracle within the contract tolerance, two resynced steps."""
    wl = synthgen.WORKLOADS["C1"].with_(rows=(64,), slot_table=(0, 0), dim=16, opt=opt, init_accum=0.0)
    cfg = O.config_from_workload(wl)
    layer = _layer(wl, 64, 128)
    ora = O.OracleEmbedding(cfg)
    rng = np.random.default_rng(7)
    try:
        rows = np.arange(64)
        w0 = (rng.standard_normal((64, 16)) * 1e-3).astype(np.float32)
        aw = 16 if opt == "adagrad" else 1
        a0 = np.where(np.arange(64)[:, None] % 3 == 0, 1e6, np.where(np.arange(64)[:, None] % 3 == 1, 1e-30, 0.5))
        a0 = np.broadcast_to(a0, (64, aw)).astype(np.float32).copy()
        layer.write_rows(0, rows, w0, a0)
        for step in range(2):
            ids = np.concatenate([np.arange(64), rng.integers(0, 8, 64)])  # slot 0: every row; slot 1: hot rows
            offs = np.arange(129)
            dy = np.empty((64, 2, 16), np.float32)
            scale = np.where(np.arange(64) % 4 == 0, 1e4, np.where(np.arange(64) % 4 == 1, 1e-40, 1.0))
            dy[:, 0, :] = (rng.standard_normal((64, 16)) * scale[:, None]).astype(np.float32)
            dy[:, 1, :] = rng.standard_normal((64, 16)).astype(np.float32)
            bt = synthgen.Batch(ids=ids.astype(np.int64), offsets=offs.astype(np.int64), batch=64, dy=dy)
            w, a = _read_global(layer, cfg, rows)
            ora.load_rows(rows, w, a)
            Y, *_ = _run_step(torch, layer, bt, lr)
            (Yo,) = ora.lookup([(bt.ids, bt.offsets, 64)])
            _check_close(Y, Yo, f"Y step {step}")
            ora.backward_update([bt.dy], lr)
            w, a = _read_global(layer, cfg, rows)
            wo, ao = ora.rows(rows)
            _check_close(w, wo, f"w step {step} lr {lr}")
            _check_close(a, ao, f"a step {step} lr {lr}")
    finally:
        layer.close()
