"""Pins for oracle.sweep: brute force on the tiny space, the all-ties net, the
affine-net closed form and sub-range merge invariance."""

import numpy as np

import workloads
from oracle import space, sweep
from tests import pins


def test_tiny_space_brute_force_times_and_full_sort():
    vl = workloads.space("tiny")
    model = workloads.random_net(vl, [4, 3], seed=5)
    ref = pins.brute_times(model, vl)
    t = sweep.times(model, vl, 0, 2 ** 14)
    assert np.max(np.abs(t - np.array(ref))) < 1e-12
    # full sort by (t, I) with Python's tuple order (independent of lexsort)
    best = sorted((tt, i) for i, tt in enumerate(ref))[:37]
    idx, tk = sweep.topk(model, vl, 37, chunk=3000)
    assert [int(i) for i in idx] == [i for _, i in best]


def test_trained_tiny_model_matches_brute_force():
    vl = workloads.space("tiny")
    model = workloads.load_model("tiny_14-32-32-1")
    ref = np.array(pins.brute_times(model, vl))
    t = sweep.times(model, vl, 0, 2 ** 14)
    assert np.max(np.abs(t - ref) / np.abs(ref)) < 1e-12
    i1, _ = sweep.topk(model, vl, 1)
    assert int(i1[0]) == int(np.argmin(ref))


def test_all_ties_net_returns_first_indices():
    vl = workloads.space("cfg2")
    model = workloads.all_ties_net(vl, [8, 8])
    idx, t = sweep.topk(model, vl, 16, begin=123456, end=123456 + 5000)
    assert [int(i) for i in idx] == list(range(123456, 123456 + 16))
    assert np.all(t == model["y_mean"] + model["y_scale"] * 0.25)


def test_affine_net_closed_form_kbest():
    vl = [[64, 128, 256, 512, 1024], [32, 64, 128]] * 5   # 15^5 = 759,375 configs
    model = workloads.affine_net(vl, [32, 32], seed=3)
    ci, ct = pins.affine_kbest(model, vl, 50)
    idx, t = sweep.topk(model, vl, 50)
    assert [int(i) for i in idx] == ci
    assert np.max(np.abs(t - np.array(ct))) < 1e-12
    # affinity really holds (no unit switches off): compare the full table on a slice
    C, tables = pins.affine_tables(model, vl)
    sl = np.arange(1000, 3000, dtype=np.uint64)
    d = space.decode(sl, [len(v) for v in vl])
    closed = C + sum(tables[j][d[:, j]] for j in range(len(vl)))
    assert np.max(np.abs(sweep.times(model, vl, 1000, 3000) - closed)) < 1e-12


def test_subrange_merge_invariance():
    vl = workloads.space("cfg2")
    model = workloads.random_net(vl, [16, 16], seed=8)
    a, b = 10_000_000, 10_060_000
    full = sweep.topk(model, vl, 25, a, b)
    parts = [sweep.topk(model, vl, 25, *space.shard(b - a, 4, r)) for r in range(0)]
    parts = []
    for r in range(4):
        lo, hi = space.shard(b - a, 4, r)
        parts.append(sweep.topk(model, vl, 25, a + lo, a + hi))
    merged = sweep.merge_topk(parts, 25)
    assert np.array_equal(full[0], merged[0]) and np.array_equal(full[1], merged[1])


def test_k_larger_than_range_and_nan_order():
    vl = workloads.space("tiny")
    model = workloads.random_net(vl, [4], seed=1)
    idx, t = sweep.topk(model, vl, 10, begin=100, end=104)
    assert len(idx) == 4 and sorted(idx.tolist()) == [100, 101, 102, 103]
    i, tt = sweep.merge_topk([(np.array([5, 3, 9], np.uint64), np.array([np.nan, np.inf, 1.0]))], 3)
    assert i.tolist() == [9, 3, 5]
