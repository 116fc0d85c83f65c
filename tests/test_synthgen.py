"""Input-generator checks (-m "not gpu"): shapes, CSR validity, determinism and the distributions the
recipe in DESIGN.md §4 promises."""
import numpy as np
import pytest

import synthgen


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5"])
def test_csr_shapes_and_ranges(name):
    wl = synthgen.WORKLOADS[name]
    bt = synthgen.make_batch(wl, batch=64)
    S = wl.num_slots
    assert bt.offsets.shape == (S * 64 + 1,) and bt.offsets[0] == 0 and np.all(np.diff(bt.offsets) >= 0)
    assert bt.ids.shape == (bt.nnz,) and bt.dy.shape == (64, S, wl.dim) and bt.dy.dtype == np.float32
    for s in range(S):
        ids = bt.ids[bt.offsets[s * 64]:bt.offsets[(s + 1) * 64]]
        assert ids.min(initial=0) >= 0 and ids.max(initial=0) < wl.rows[wl.slot_table[s]]
    assert np.all(bt.dy >= -1) and np.all(bt.dy < 1)


def test_deterministic_and_rank_step_distinct():
    wl = synthgen.WORKLOADS["C2"]
    a = synthgen.make_batch(wl, rank=0, step=0, batch=128)
    b = synthgen.make_batch(wl, rank=0, step=0, batch=128)
    c = synthgen.make_batch(wl, rank=1, step=0, batch=128)
    assert np.array_equal(a.ids, b.ids) and np.array_equal(a.dy, b.dy)
    assert not np.array_equal(a.ids, c.ids)


def test_zipf_unique_fraction_matches_appendix_b():
    # C2 per table E[U] = 7,820 of 16,384 draws (Monte-Carlo 7,812)
    wl = synthgen.WORKLOADS["C2"]
    rng = np.random.default_rng(0)
    ids = synthgen.draw_ids(wl, rng, 0, 16384)
    assert abs(np.unique(ids).size - 7820) < 200


def test_hot1k_fraction():
    wl = synthgen.WORKLOADS["C5"]
    rng = np.random.default_rng(1)
    ids = synthgen.draw_ids(wl, rng, 3, 200000)
    hot = synthgen.permute_rank(np.arange(1, 1001), wl.rows[3], 3)
    frac = np.isin(ids, hot).mean()
    assert 0.89 < frac < 0.91


def test_permutation_is_bijective():
    R = 10007 * 3
    k = np.arange(1, R + 1)
    assert np.unique(synthgen.permute_rank(k, R, 5)).size == R
