"""W > 1 parity on ANY number of GPUs (-m gpu): all W ranks of the row-sharded layer live in this
process (emb_create_group); on a one-GPU box they are emulated on cuda:0. The exchange kernels are the
ones a one-process-per-GPU rank runs (route -> peer key stores, owner merge tree, peer-load pull of the
remote rows, requester gradient merge -> peer stores into the owners' regions, owner merge + apply); the
group calls order the ranks' phases with cross-stream events so no kernel ever waits on a kernel that is
not already complete. Checks per step: see tests/mrank_cases.py."""
import numpy as np
import pytest

import synthgen
from oracle import emb_oracle as O
import mrank_cases as C  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    t = pytest.importorskip("torch")
    if not t.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2112_02752_b200 import build
    build.build()
    return t


def _device_batches(batches, wl, devices):
    from paper_2112_02752_b200.harness import DeviceBatch
    return [DeviceBatch(b, wl.num_slots, wl.dim, devices[r]) for r, b in enumerate(batches)]


def _step(grp, dbs, lr, torch):
    grp.lookup([d.ids for d in dbs], [d.offsets for d in dbs], [d.batch for d in dbs], [d.nnz for d in dbs],
               [d.out for d in dbs])
    torch.cuda.synchronize()


def _run_group(torch, case, world, shard="cyclic", devices=None, prefetch=False):
    from paper_2112_02752_b200.harness import make_group
    devices = devices or [0] * world
    wl, B, steps = C.case_workload(case, world)
    cfgW = O.config_from_workload(wl, world=world, shard=shard)
    cfg1 = O.config_from_workload(wl, world=1)
    bts = [[C.case_batch(case, wl, B, r, s) for r in range(world)] for s in range(steps)]
    max_ids = [max(max(bts[s][r].nnz for s in range(steps)), 1) for r in range(world)]
    grp = make_group(wl, world=world, max_batch=B + 16 * world, max_ids=max_ids, devices=devices, shard=shard)
    ora = O.OracleEmbedding(cfg1)
    msgs = []
    all_dbs = [_device_batches(bts[s], wl, devices) for s in range(steps)]
    try:
        for s in range(steps):
            batches = bts[s]
            owned = [C.owned_touched(cfg1, cfgW, batches, r) for r in range(world)]
            for r in range(world):  # stepwise resync (R22): the GPU's pre-step state of every touched row
                mine, t_of = owned[r]
                if mine.size:
                    ora.load_rows(mine, *C.read_owned(grp.layers[r], cfg1, mine, t_of, wl.dim))
            dbs = all_dbs[s]
            _step(grp, dbs, wl.lr, torch)
            Yo = ora.lookup([(b.ids, b.offsets, b.batch) for b in batches])
            infos = [l.step_info() for l in grp.layers]
            for r in range(world):
                lay = grp.layers[r]
                keys, counts = lay.last_unique()
                okeys, fanin = lay.last_owner_unique()
                C.check_rank_step(msgs, s, r, cfgW, ora, batches, dbs[r].out.cpu().numpy(), Yo[r], infos[r], keys,
                                  counts, okeys, fanin, [infos[q]["send_counts"][r] for q in range(world)])
            if prefetch and s + 1 < steps:  # the next step's sort + route overlaps this backward
                nx = all_dbs[s + 1]
                grp.lookup_prefetch([d.ids for d in nx], [d.offsets for d in nx], [d.batch for d in nx],
                                    [d.nnz for d in nx])
            grp.backward_update([d.dy for d in dbs], wl.lr)
            torch.cuda.synchronize()
            ora.backward_update([b.dy for b in batches], wl.lr)
            for r in range(world):
                mine, t_of = owned[r]
                w, a = C.read_owned(grp.layers[r], cfg1, mine, t_of, wl.dim)
                wo, ao = ora.rows(mine)
                if not C.close(w, wo):
                    msgs.append(f"step {s} rank {r}: updated w mismatch (max err {np.abs(w - wo).max():.3g})")
                if wl.opt != "sgd" and not C.close(a, ao):
                    msgs.append(f"step {s} rank {r}: updated a mismatch")
    finally:
        grp.close()
    assert not msgs, "\n".join(msgs)


@pytest.mark.parametrize("case,world,shard", [
    ("c3", 2, "cyclic"), ("c3", 4, "cyclic"), ("c3", 2, "block"), ("c3", 3, "block"),
    ("hot", 2, "cyclic"), ("hot", 4, "block"), ("c3rw", 2, "cyclic"), ("c3rw", 4, "cyclic"),
    ("gen", 2, "cyclic"), ("gen", 4, "cyclic"), ("edge", 2, "cyclic"), ("edge", 4, "block"),
    ("c5", 2, "cyclic"), ("c3full", 2, "cyclic"), ("c3full", 4, "cyclic"),
    # W = 8 (BJ:9-11's GPU count) and 16 (EMB_MAX_WORLD) emulated on one GPU: 3- and 4-pass merge
    # trees, 8- / 16-way regions and flags
    ("c3", 8, "cyclic"), ("hot", 8, "block"), ("gen", 8, "cyclic"), ("c3rw", 8, "cyclic"), ("c3", 16, "cyclic"),
    ("skew", 2, "cyclic")])
def test_group_row_sharded_parity(torch, case, world, shard):
    _run_group(torch, case, world, shard)


@pytest.mark.parametrize("case,world,shard", [
    ("c3", 2, "cyclic"), ("c3", 4, "block"), ("hot", 3, "cyclic"), ("c3rw", 2, "cyclic"), ("edge", 2, "cyclic"),
    ("edge", 4, "block"), ("gen", 2, "cyclic"), ("c3full", 2, "cyclic"), ("c3", 8, "cyclic")])
def test_group_prefetch_parity(torch, case, world, shard):
    """emb_lookup_prefetch_group before every backward: the next step's sort + route (keys already in
    the owners' regions, buffer set epoch & 1) overlaps this step's gradient passes; results as without."""
    _run_group(torch, case, world, shard, prefetch=True)


def test_group_prefetch_mismatch_and_state(torch):
    """A lookup whose arguments differ from the pending prefetch takes part with an empty batch and fails
    the step on every rank (no row changes anywhere); a second prefetch before the lookup is a state
    error; afterwards plain and prefetched steps match the oracle again."""
    from paper_2112_02752_b200.emb import EmbError, EMB_ERR_INVALID, EMB_ERR_STATE
    from paper_2112_02752_b200.harness import make_group
    W = 2
    wl = synthgen.WORKLOADS["C3"].with_(rows=(4000, 3000), slot_table=(0, 1), dim=16, opt="adagrad")
    cfgW = O.config_from_workload(wl, world=W)
    cfg1 = O.config_from_workload(wl, world=1)
    B = 64
    bts = [[synthgen.make_batch(wl, rank=r, step=s, batch=B) for r in range(W)] for s in range(4)]
    grp = make_group(wl, world=W, max_batch=B, max_ids=max(b.nnz for st in bts for b in st))
    try:
        all_rows = [np.arange(O.rows_local(cfgW, r)) for r in range(W)]

        def snapshot():
            out = []
            for r in range(W):
                g = all_rows[r] * W + r  # cyclic: local -> global
                t = np.searchsorted(cfg1.base, g, side="right") - 1
                out.append(C.read_owned(grp.layers[r], cfg1, g, t, wl.dim))
            return out

        dbs = [_device_batches(bts[s], wl, [0] * W) for s in range(4)]
        pf = lambda d: grp.lookup_prefetch([x.ids for x in d], [x.offsets for x in d],  # noqa: E731
                                           [x.batch for x in d], [x.nnz for x in d])
        # a request with no backward before the lookup launched nothing: dropped, the lookup is plain
        ora = O.OracleEmbedding(cfg1)
        pf(dbs[1])
        with pytest.raises(EmbError) as ei:
            pf(dbs[1])
        assert ei.value.status == EMB_ERR_STATE
        _step(grp, dbs[0], wl.lr, torch)
        Yo = ora.lookup([(b.ids, b.offsets, b.batch) for b in bts[0]])
        for r in range(W):
            assert C.close(dbs[0][r].out.cpu().numpy(), Yo[r]), f"step 0 rank {r}: Y mismatch"
        # prefetch step 1, launched by step 0's backward; then rank 1 looks up other inputs
        pf(dbs[1])
        grp.backward_update([d.dy for d in dbs[0]], wl.lr)
        torch.cuda.synchronize()
        before = snapshot()
        mixed = [dbs[1][0], dbs[2][1]]
        with pytest.raises(EmbError) as ei:
            _step(grp, mixed, wl.lr, torch)
        assert ei.value.status == EMB_ERR_INVALID
        with pytest.raises(EmbError):
            grp.backward_update([d.dy for d in mixed], wl.lr)
        torch.cuda.synchronize()
        after = snapshot()
        for r in range(W):
            assert np.array_equal(before[r][0], after[r][0]) and np.array_equal(before[r][1], after[r][1]), \
                f"rank {r} changed rows in an aborted step"
        for r in range(W):
            grp.layers[r].clear_error()
        # steps 2 (plain) and 3 (prefetched during step 2's backward) match the oracle
        ora = O.OracleEmbedding(cfg1)
        for r in range(W):  # (resync: the oracle starts from the GPU's state after step 0)
            mine = np.concatenate([C.owned_touched(cfg1, cfgW, bts[s], r)[0] for s in (2, 3)])
            mine = np.unique(mine)
            if mine.size:
                t_of = np.searchsorted(cfg1.base, mine, side="right") - 1
                ora.load_rows(mine, *C.read_owned(grp.layers[r], cfg1, mine, t_of, wl.dim))
        for s in (2, 3):
            _step(grp, dbs[s], wl.lr, torch)
            Yo = ora.lookup([(b.ids, b.offsets, b.batch) for b in bts[s]])
            for r in range(W):
                assert C.close(dbs[s][r].out.cpu().numpy(), Yo[r]), f"step {s} rank {r}: Y mismatch"
            if s == 2:
                grp.lookup_prefetch([d.ids for d in dbs[3]], [d.offsets for d in dbs[3]], [d.batch for d in dbs[3]],
                                    [d.nnz for d in dbs[3]])
            grp.backward_update([d.dy for d in dbs[s]], wl.lr)
            torch.cuda.synchronize()
            ora.backward_update([b.dy for b in bts[s]], wl.lr)
            for r in range(W):
                mine, t_of = C.owned_touched(cfg1, cfgW, bts[s], r)
                w, a = C.read_owned(grp.layers[r], cfg1, mine, t_of, wl.dim)
                assert C.close(w, ora.rows(mine)[0]) and C.close(a, ora.rows(mine)[1]), f"step {s} rank {r}"
    finally:
        grp.close()


def test_group_on_distinct_devices(torch):
    """The same group mode with each rank on its own GPU (peer access between devices)."""
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs 2 GPUs")
    W = min(n, 4)
    _run_group(torch, "c3", W, "cyclic", devices=list(range(W)))


def test_group_input_error_aborts_every_rank(torch):
    """An out-of-range id on rank 1 (step 0) and bad arguments on rank 0 (step 1): both steps take part
    collectively, update no row on any rank, the valid bags' Y are still right, the errors are reported,
    and after emb_clear_error the next step matches the oracle again."""
    from paper_2112_02752_b200.emb import EmbError, EMB_ERR_INVALID, EMB_ERR_RANGE
    from paper_2112_02752_b200.harness import make_group
    W = 2
    wl = synthgen.WORKLOADS["C3"].with_(rows=(4000, 3000), slot_table=(0, 1), dim=16, opt="adagrad")
    cfgW = O.config_from_workload(wl, world=W)
    cfg1 = O.config_from_workload(wl, world=1)
    B = 64
    bts = [[synthgen.make_batch(wl, rank=r, step=s, batch=B) for r in range(W)] for s in range(3)]
    bad_ids = bts[0][1].ids.copy()
    bad_ids[5] = 4000 + 17  # slot 0 -> table 0 has 4000 rows
    bts[0][1] = synthgen.Batch(ids=bad_ids, offsets=bts[0][1].offsets, batch=B, dy=bts[0][1].dy)
    grp = make_group(wl, world=W, max_batch=B, max_ids=max(b.nnz for st in bts for b in st))
    try:
        all_rows = [np.arange(O.rows_local(cfgW, r)) for r in range(W)]

        def snapshot():
            out = []
            for r in range(W):
                g = all_rows[r] * W + r  # cyclic: local -> global
                t = np.searchsorted(cfg1.base, g, side="right") - 1
                out.append(C.read_owned(grp.layers[r], cfg1, g, t, wl.dim))
            return out

        before = snapshot()
        dbs = _device_batches(bts[0], wl, [0] * W)
        try:
            _step(grp, dbs, wl.lr, torch)
        except EmbError:
            pass  # the error may already be visible to the host here
        with pytest.raises(EmbError) as ei:
            grp.backward_update([d.dy for d in dbs], wl.lr)
        assert ei.value.status == EMB_ERR_RANGE
        torch.cuda.synchronize()
        # rank 0's bags are all valid: its Y equals the oracle on the pre-step state
        ora = O.OracleEmbedding(cfg1)
        b0 = bts[0][0]
        (Y0,) = ora.lookup([(b0.ids, b0.offsets, b0.batch)])
        assert C.close(dbs[0].out.cpu().numpy(), Y0)
        after = snapshot()
        for r in range(W):
            assert np.array_equal(before[r][0], after[r][0]) and np.array_equal(before[r][1], after[r][1]), \
                f"rank {r} changed rows in an aborted step"
        grp.layers[1].clear_error()
        # step 1: bad arguments on rank 0 (nnz above capacity): it takes part with an empty batch
        dbs = _device_batches(bts[1], wl, [0] * W)
        with pytest.raises(EmbError) as ei:
            grp.lookup([d.ids for d in dbs], [d.offsets for d in dbs], [d.batch for d in dbs],
                       [10 ** 6, dbs[1].nnz], [d.out for d in dbs])
        assert ei.value.status == EMB_ERR_INVALID
        with pytest.raises(EmbError):
            grp.backward_update([d.dy for d in dbs], wl.lr)
        torch.cuda.synchronize()
        after2 = snapshot()
        for r in range(W):
            assert np.array_equal(before[r][0], after2[r][0]), f"rank {r} changed rows in an aborted step"
        grp.layers[0].clear_error()
        # step 2: clean again -> matches the oracle (started from the unchanged initial state)
        dbs = _device_batches(bts[2], wl, [0] * W)
        _step(grp, dbs, wl.lr, torch)
        grp.backward_update([d.dy for d in dbs], wl.lr)
        torch.cuda.synchronize()
        ora = O.OracleEmbedding(cfg1)
        Yo = ora.lookup([(b.ids, b.offsets, b.batch) for b in bts[2]])
        for r in range(W):
            assert C.close(dbs[r].out.cpu().numpy(), Yo[r])
        ora.backward_update([b.dy for b in bts[2]], wl.lr)
        for r in range(W):
            mine, t_of = C.owned_touched(cfg1, cfgW, bts[2], r)
            w, a = C.read_owned(grp.layers[r], cfg1, mine, t_of, wl.dim)
            assert C.close(w, ora.rows(mine)[0]) and C.close(a, ora.rows(mine)[1])
    finally:
        grp.close()


def test_group_bitwise_determinism(torch):
    """Two runs of the same 2-rank group give bitwise identical Y and rows (fixed merge orders, R10)."""
    from paper_2112_02752_b200.harness import make_group
    W = 2
    wl = synthgen.WORKLOADS["C5"].with_(rows=(200_000,) * 4, slot_table=(0, 1, 2, 3), bag_len=16)
    bts = [[synthgen.make_batch(wl, rank=r, step=s, batch=256) for r in range(W)] for s in range(2)]
    res = []
    for _ in range(2):
        grp = make_group(wl, world=W, max_batch=256, max_ids=max(b.nnz for st in bts for b in st))
        Ys = []
        for s in range(2):
            dbs = _device_batches(bts[s], wl, [0] * W)
            _step(grp, dbs, wl.lr, torch)
            grp.backward_update([d.dy for d in dbs], wl.lr)
            torch.cuda.synchronize()
            Ys.append([d.out.cpu().numpy() for d in dbs])
        # table 1 starts at g = 200,000 (even): cyclic owner = id mod 2
        rows = [grp.layers[r].read_rows(1, np.arange(r, 200_000, 14)) for r in range(W)]
        res.append((Ys, rows))
        grp.close()
    for ya, yb in zip(res[0][0], res[1][0]):
        for a, b in zip(ya, yb):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    for (wa, aa), (wb, ab) in zip(res[0][1], res[1][1]):
        assert np.array_equal(wa.view(np.uint32), wb.view(np.uint32))
        assert np.array_equal(aa.view(np.uint32), ab.view(np.uint32))
