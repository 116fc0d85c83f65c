"""Pins for the CPU oracle (-m "not gpu"). Each test ties an oracle function to something other than
itself: a hand-worked example (tests/golden/), a published test vector, a textbook/library routine
(dense one-hot matmul, torch CPU EmbeddingBag + torch.optim), brute force on tiny inputs, or an
invariant. See DESIGN.md §5 for the pin table."""
import json
import os
from collections import Counter

import numpy as np
import pytest

from oracle import emb_oracle as O
import synthgen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------------------- init hash (R15)
def test_splitmix64_published_vectors():
    # SplitMix64 reference outputs for seed 1234567 (the test vector shipped with the public
    # xoshiro/splitmix64 reference code and reproduced by e.g. Rust rand_xoshiro's SplitMix64 test),
    # and the well-known first output for seed 0 (0xE220A8397B1DCDAF).
    expect = [6457827717110365317, 3203168211198807973, 9817491932198370423,
              4593380528125082431, 16408922859458223821]
    state = 1234567
    got = []
    for _ in range(5):
        got.append(int(O.splitmix64_next(np.array([state], dtype=np.uint64))[0]))
        state = (state + 0x9E3779B97F4A7C15) & O.MASK64
    assert got == expect
    assert int(O.splitmix64_next(np.array([0], dtype=np.uint64))[0]) == 0xE220A8397B1DCDAF


def test_init_weights_definition_and_range():
    # w = int16(h >> 48) * 2^-19: brute-force one element with Python ints, check the range and exactness
    seed, D = 2112, 8
    g = np.array([0, 1, 12345, 10**9 - 1], dtype=np.int64)
    w = O.init_weights(seed, g, D)
    for i, gi in enumerate(g):
        for c in range(D):
            x = seed ^ (int(gi) * D + c)
            z = (x + 0x9E3779B97F4A7C15) & O.MASK64
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & O.MASK64
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & O.MASK64
            z ^= z >> 31
            top = z >> 48
            top = top - 65536 if top >= 32768 else top
            assert w[i, c] == np.float32(top / 2.0 ** 19)
    big = O.init_weights(7, np.arange(20000), 16)
    assert big.min() >= -1 / 16 and big.max() < 1 / 16
    assert abs(float(big.mean())) < 1e-3
    # every value is an integer multiple of 2^-19 (exact in fp32)
    assert np.all(np.round(big.astype(np.float64) * 2 ** 19) == big.astype(np.float64) * 2 ** 19)


# ----------------------------------------------------------------------------- worked example
def _worked_cfg(pool, world=1, shard="cyclic"):
    d = _gold("worked_example.json")
    cfg = O.OracleConfig(rows=tuple(d["rows"]), dim=d["dim"], slot_table=tuple(d["slot_table"]), pool=pool,
                         opt="sgd", world=world, shard=shard)
    return d, cfg


@pytest.mark.parametrize("pool", ["sum", "mean"])
def test_worked_example_forward_backward_sgd(pool):
    d, cfg = _worked_cfg(pool)
    emb = O.OracleEmbedding(cfg)
    table = np.array(d["table"], dtype=np.float32)
    emb.load_rows(np.arange(4), table, np.zeros_like(table))
    ids, offs, B = np.array(d["ids"]), np.array(d["offsets"]), d["batch"]
    (Y,) = emb.lookup([(ids, offs, B)])
    np.testing.assert_array_equal(Y, np.array(d[pool]["Y"], dtype=np.float32))
    dy = np.ones((B, 2, 2), dtype=np.float32)
    U, G = O.merged_grads(cfg, [(ids, offs, B, dy)])
    np.testing.assert_array_equal(U, d["unique"])
    gcol = np.zeros(4)
    gcol[U] = G[:, 0]
    np.testing.assert_array_equal(gcol, d[pool]["G_col"])
    emb.backward_update([dy], d["lr"])
    w, _ = emb.rows(np.arange(4))
    np.testing.assert_array_equal(w, np.array(d[pool]["table_after_sgd"], dtype=np.float32))


def test_worked_example_dedup_and_routing():
    d, cfg = _worked_cfg("sum", world=2)
    ids, offs, B = np.array(d["ids"]), np.array(d["offsets"]), d["batch"]
    g, _, _ = O.occurrence_keys(cfg, ids, offs, B)
    U, counts, inv = O.dedup(g)
    assert U.tolist() == d["unique"] and counts.tolist() == d["counts"]
    lists, cnt = O.route(cfg, U)
    assert lists[0].tolist() == d["route_w2_cyclic"]["to_rank0"]
    assert lists[1].tolist() == d["route_w2_cyclic"]["to_rank1"]
    _, cfgb = _worked_cfg("sum", world=2, shard="block")
    lists, _ = O.route(cfgb, U)
    assert lists[0].tolist() == d["route_w2_block"]["to_rank0"]
    assert lists[1].tolist() == d["route_w2_block"]["to_rank1"]


def test_adagrad_hand_worked():
    d = _gold("adagrad_hand.json")
    cfg = O.OracleConfig(rows=(1,), dim=1, slot_table=(0,), pool="sum", opt="adagrad", eps=d["eps"])
    emb = O.OracleEmbedding(cfg)
    emb.load_rows(np.array([0]), np.array([[d["w0"]]], np.float32), np.array([[d["a0"]]], np.float32))
    for st in d["steps"]:
        occ = st["occurrences"]
        ids = np.zeros(len(occ), dtype=np.int64)
        offs = np.arange(len(occ) + 1)  # one bag per occurrence, each holding row 0
        emb.lookup([(ids, offs, len(occ))])
        dy = np.array(occ, dtype=np.float32).reshape(len(occ), 1, 1)
        emb.backward_update([dy], d["lr"])
        w, a = emb.rows(np.array([0]))
        assert a[0, 0] == np.float32(st["a"])
        assert w[0, 0] == np.float32(st["w"])


def test_rowwise_adagrad_hand_worked():
    # SURVEY §8(f) f1 / reading R14': hand-worked fixture (exact binary-fraction inputs)
    d = _gold("rowwise_adagrad_hand.json")
    cfg = O.OracleConfig(rows=(1,), dim=2, slot_table=(0,), pool="sum", opt="rowwise_adagrad", eps=d["eps"])
    emb = O.OracleEmbedding(cfg)
    emb.load_rows(np.array([0]), np.array([d["w0"]], np.float32), np.array([[d["a0"]]], np.float32))
    for st in d["steps"]:
        occ = st["occurrences"]
        ids = np.zeros(len(occ), dtype=np.int64)
        offs = np.arange(len(occ) + 1)
        emb.lookup([(ids, offs, len(occ))])
        dy = np.array(occ, dtype=np.float32).reshape(len(occ), 1, 2)
        emb.backward_update([dy], d["lr"])
        w, a = emb.rows(np.array([0]))
        assert a.shape == (1, 1)
        assert a[0, 0] == np.float32(st["a"])
        assert np.array_equal(w[0], np.array(st["w_fp64"], dtype=np.float32))


def test_rowwise_adagrad_reduces_to_elementwise():
    # special cases that reduce to the (torch-pinned) element-wise Adagrad: D = 1, and a gradient whose
    # columns are all equal (mean_c G^2 = G^2 in every column) with equal initial accumulators
    rng = np.random.default_rng(5)
    for D, equal_cols in ((1, False), (8, True)):
        U = 50
        w = rng.standard_normal((U, D)).astype(np.float32)
        a0 = rng.uniform(0, 2, (U, 1)).astype(np.float32)
        G = rng.standard_normal((U, 1 if equal_cols else D)) * np.ones((1, D))
        w_r, a_r = O.rowwise_adagrad_update(w, a0, G, 0.05, 1e-6)
        w_e, a_e = O.adagrad_update(w, np.repeat(a0, D, axis=1), G, 0.05, 1e-6)
        assert np.array_equal(w_r, w_e)
        assert np.array_equal(np.repeat(a_r, D, axis=1), a_e)


def test_rowwise_adagrad_state_is_per_row_and_monotone():
    cfg = O.OracleConfig(rows=(40,), dim=4, slot_table=(0,), opt="rowwise_adagrad", init_accum=0.1)
    emb = O.OracleEmbedding(cfg)
    ids = np.array([3, 3, 7, 11], dtype=np.int64)
    offs = np.array([0, 2, 3, 4])
    prev = emb.rows(np.array([3, 7, 11, 20]))[1]
    assert prev.shape == (4, 1) and np.all(prev == np.float32(0.1))
    emb.lookup([(ids, offs, 3)])
    emb.backward_update([np.ones((3, 1, 4), np.float32)], 0.01)
    w, a = emb.rows(np.array([3, 7, 11, 20]))
    # row 3: two occurrences of an all-ones dY -> G = 2 in every column -> a = 0.1 + 4
    assert a[0, 0] == np.float32(np.float64(np.float32(0.1)) + 4.0)
    assert a[1, 0] == a[2, 0] == np.float32(np.float64(np.float32(0.1)) + 1.0)
    assert a[3, 0] == np.float32(0.1)  # untouched
    assert np.array_equal(w[3], O.init_weights(cfg.seed, np.array([20]), 4)[0])


# ----------------------------------------------------------------------------- dense one-hot matmul
def _onehot(cfg, ids, offs, B, s):
    """A_s[b, id] = multiplicity of id in bag (s, b) — built by a plain Python loop (brute force)."""
    R = cfg.rows[cfg.slot_table[s]]
    A = np.zeros((B, R))
    for b in range(B):
        for j in range(offs[s * B + b], offs[s * B + b + 1]):
            A[b, ids[j]] += 1
    return A


@pytest.mark.parametrize("pool", ["sum", "mean"])
def test_pooling_equals_dense_onehot_matmul(pool):
    wl = synthgen.WORKLOADS["C1"].with_(rows=(300, 200), slot_table=(0, 1, 0), pool=pool, dim=8)
    cfg = O.config_from_workload(wl)
    bt = synthgen.make_batch(wl, batch=37, empty_frac=0.15)
    emb = O.OracleEmbedding(cfg)
    (Y,) = emb.lookup([(bt.ids, bt.offsets, bt.batch)])
    for s in range(len(cfg.slot_table)):
        t = cfg.slot_table[s]
        Wt = O.init_weights(cfg.seed, cfg.base[t] + np.arange(cfg.rows[t]), cfg.dim).astype(np.float64)
        A = _onehot(cfg, bt.ids, bt.offsets, bt.batch, s)
        if pool == "mean":
            L = A.sum(1)
            A = A / np.where(L > 0, L, 1)[:, None]
        ref = (A @ Wt).astype(np.float32)
        np.testing.assert_allclose(Y[:, s, :], ref, rtol=0, atol=1e-7)


@pytest.mark.parametrize("pool", ["sum", "mean"])
def test_merged_grads_equal_dense_transpose_matmul(pool):
    wl = synthgen.WORKLOADS["C1"].with_(rows=(50, 40), slot_table=(0, 1, 1), pool=pool, dim=4)
    cfg = O.config_from_workload(wl)
    bt = synthgen.make_batch(wl, batch=23, empty_frac=0.1)
    U, G = O.merged_grads(cfg, [(bt.ids, bt.offsets, bt.batch, bt.dy)])
    dense = np.zeros((cfg.total_rows, cfg.dim))
    for s in range(len(cfg.slot_table)):
        t = cfg.slot_table[s]
        A = _onehot(cfg, bt.ids, bt.offsets, bt.batch, s)
        if pool == "mean":
            L = A.sum(1)
            A = A / np.where(L > 0, L, 1)[:, None]
        dense[cfg.base[t]:cfg.base[t] + cfg.rows[t]] += A.T @ bt.dy[:, s, :].astype(np.float64)
    touched = np.zeros(cfg.total_rows, bool)
    touched[U] = True
    np.testing.assert_allclose(G, dense[U], rtol=1e-12, atol=1e-12)
    assert np.all(dense[~touched] == 0)


# ----------------------------------------------------------------------------- torch CPU cross-check
def _torch_run(cfg, batches, lr, steps_opt):
    torch = pytest.importorskip("torch")
    tabs = []
    for t, R in enumerate(cfg.rows):
        w0 = O.init_weights(cfg.seed, cfg.base[t] + np.arange(R), cfg.dim).astype(np.float64)
        tabs.append(torch.nn.Parameter(torch.tensor(w0)))
    if cfg.opt == "sgd":
        opt = torch.optim.SGD(tabs, lr=lr)
    else:
        opt = torch.optim.Adagrad(tabs, lr=lr, eps=cfg.eps, initial_accumulator_value=cfg.init_accum)
    outs = []
    for bt in batches:
        opt.zero_grad()
        B = bt.batch
        loss = 0
        Y = []
        for s, t in enumerate(cfg.slot_table):
            lo, hi = bt.offsets[s * B], bt.offsets[(s + 1) * B]
            ids = torch.tensor(bt.ids[lo:hi])
            offs = torch.tensor(bt.offsets[s * B:(s + 1) * B + 1] - lo)
            y = torch.nn.functional.embedding_bag(ids, tabs[t], offs, mode=cfg.pool, include_last_offset=True)
            Y.append(y)
            loss = loss + (y * torch.tensor(bt.dy[:, s, :].astype(np.float64))).sum()
        loss.backward()
        opt.step()
        outs.append(torch.stack(Y, 1).detach().numpy())
    return outs, [p.detach().numpy() for p in tabs], opt


@pytest.mark.parametrize("pool,opt", [("sum", "adagrad"), ("mean", "adagrad"), ("sum", "sgd"), ("mean", "sgd")])
def test_whole_step_matches_torch_cpu(pool, opt):
    wl = synthgen.WORKLOADS["C1"].with_(rows=(120, 90), slot_table=(0, 1, 0), pool=pool, opt=opt, dim=8, ids="zipf",
                                        zipf_s=1.2)
    cfg = O.config_from_workload(wl)
    lr = 0.05
    batches = [synthgen.make_batch(wl, step=k, batch=41, empty_frac=0.1) for k in range(3)]
    touts, ttabs, _ = _torch_run(cfg, batches, lr, 3)
    emb = O.OracleEmbedding(cfg)
    for k, bt in enumerate(batches):
        (Y,) = emb.lookup([(bt.ids, bt.offsets, bt.batch)])
        # torch keeps fp64 state; the oracle rounds the state to fp32 each step (R16): ~1e-7 relative
        np.testing.assert_allclose(Y, touts[k], rtol=2e-6, atol=1e-7)
        emb.backward_update([bt.dy], lr)
    for t, R in enumerate(cfg.rows):
        w, _ = emb.rows(cfg.base[t] + np.arange(R))
        np.testing.assert_allclose(w, ttabs[t], rtol=2e-6, atol=1e-7)


def test_untouched_rows_bitwise_unchanged():
    wl = synthgen.WORKLOADS["C1"].with_(rows=(5000,), dim=4)
    cfg = O.config_from_workload(wl)
    bt = synthgen.make_batch(wl, batch=16)
    emb = O.OracleEmbedding(cfg)
    emb.lookup([(bt.ids, bt.offsets, bt.batch)])
    U = emb.backward_update([bt.dy], 0.1)
    rest = np.setdiff1d(np.arange(5000), U)
    w, a = emb.rows(rest)
    assert np.array_equal(w, O.init_weights(cfg.seed, rest, 4))
    assert np.all(a == cfg.init_accum)


# ----------------------------------------------------------------------------- dedup / routing brute force
def test_dedup_brute_force_and_invariants():
    rng = np.random.default_rng(5)
    g = rng.integers(0, 40, size=300)
    U, counts, inv = O.dedup(g)
    c = Counter(g.tolist())
    assert U.tolist() == sorted(c)
    assert counts.tolist() == [c[k] for k in sorted(c)]
    assert np.all(U[inv] == g) and counts.sum() == g.size and np.all(np.diff(U) > 0)


@pytest.mark.parametrize("shard", ["cyclic", "block"])
@pytest.mark.parametrize("W", [1, 2, 3, 8])
def test_routing_closed_form_and_partition(W, shard):
    cfg = O.OracleConfig(rows=(37, 50), dim=2, slot_table=(0, 1), world=W, shard=shard)
    R = cfg.total_rows
    g = np.arange(R)
    owner, local = O.owner_local(cfg, g)
    rows_per = -(-R // W)
    for gi in range(R):  # closed form, element by element
        if shard == "cyclic":
            assert owner[gi] == gi % W and local[gi] == gi // W
        else:
            assert owner[gi] == gi // rows_per and local[gi] == gi % rows_per
    # partition of unity: every row owned exactly once, local ids dense per owner
    for r in range(W):
        mine = local[owner == r]
        assert sorted(mine.tolist()) == list(range(O.rows_local(cfg, r)))
    assert sum(O.rows_local(cfg, r) for r in range(W)) == R
    rng = np.random.default_rng(W)
    U = np.unique(rng.integers(0, R, size=40))
    lists, cnt = O.route(cfg, U)
    assert cnt.sum() == U.size
    assert np.array_equal(np.sort(np.concatenate(lists)), U)
    for d, lst in enumerate(lists):
        assert np.all(np.diff(lst) > 0) and np.all(O.owner_local(cfg, lst)[0] == d)


def test_owner_sets_counts_equal_global_counts():
    wl = synthgen.WORKLOADS["C1"].with_(rows=(400,), dim=4, ids="zipf", zipf_s=1.1)
    W = 3
    cfg = O.config_from_workload(wl, world=W)
    per_U, per_c, all_g = [], [], []
    for r in range(W):
        bt = synthgen.make_batch(wl, rank=r, batch=20)
        g, _, _ = O.occurrence_keys(cfg, bt.ids, bt.offsets, bt.batch)
        U, c, _ = O.dedup(g)
        per_U.append(U)
        per_c.append(c)
        all_g.append(g)
    Ug, cg, _ = O.dedup(np.concatenate(all_g))
    sets = O.owner_sets(cfg, per_U, per_c)
    merged_U = np.concatenate([s[0] for s in sets])
    merged_c = np.concatenate([s[1] for s in sets])
    order = np.argsort(merged_U)
    assert np.array_equal(merged_U[order], Ug) and np.array_equal(merged_c[order], cg)


# ----------------------------------------------------------------------------- W ranks == 1 rank
@pytest.mark.parametrize("W", [2, 3])
def test_w_ranks_equal_one_rank_on_concatenated_batch(W):
    wl = synthgen.WORKLOADS["C1"].with_(rows=(700, 300), slot_table=(0, 1), dim=4, ids="zipf", zipf_s=1.1,
                                        opt="adagrad")
    cfgW = O.config_from_workload(wl, world=W)
    cfg1 = O.config_from_workload(wl, world=1)
    embW, emb1 = O.OracleEmbedding(cfgW), O.OracleEmbedding(cfg1)
    for step in range(2):
        bts = [synthgen.make_batch(wl, rank=r, step=step, batch=9 + r) for r in range(W)]
        # concatenate along the batch axis (slot-major CSR has to be re-interleaved per slot)
        S = len(wl.slot_table)
        ids, lens, dys = [], [], []
        for s in range(S):
            for bt in bts:
                lo, hi = bt.offsets[s * bt.batch], bt.offsets[(s + 1) * bt.batch]
                ids.append(bt.ids[lo:hi])
                lens.append(np.diff(bt.offsets[s * bt.batch:(s + 1) * bt.batch + 1]))
        Bt = sum(bt.batch for bt in bts)
        offs = np.concatenate([[0], np.cumsum(np.concatenate(lens))])
        YW = embW.lookup([(bt.ids, bt.offsets, bt.batch) for bt in bts])
        (Y1,) = emb1.lookup([(np.concatenate(ids), offs, Bt)])
        np.testing.assert_array_equal(np.concatenate(YW, 0), Y1)
        embW.backward_update([bt.dy for bt in bts], 0.1)
        emb1.backward_update([np.concatenate([bt.dy for bt in bts], 0)], 0.1)
        g = np.arange(cfg1.total_rows)
        np.testing.assert_allclose(embW.rows(g)[0], emb1.rows(g)[0], rtol=1e-7, atol=0)


def test_invalid_inputs_raise():
    cfg = O.OracleConfig(rows=(10,), dim=2, slot_table=(0,))
    with pytest.raises(ValueError):
        O.occurrence_keys(cfg, np.array([10]), np.array([0, 1]), 1)
    with pytest.raises(ValueError):
        O.occurrence_keys(cfg, np.array([-1]), np.array([0, 1]), 1)
    with pytest.raises(ValueError):
        O.occurrence_keys(cfg, np.array([1, 2]), np.array([0, 2, 1]), 2)
