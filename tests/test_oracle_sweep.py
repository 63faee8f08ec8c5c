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


def _combined_net(value_lists, n_const, seed):
    """A random F-input net (F = P + n_const) whose scaler moves and scales every
    column, device columns included (shift != 0, scale != 1), so that a device
    feature left unscaled, or prepended instead of appended, changes t."""
    ext = [list(v) for v in value_lists] + [[0.0, 1.0]] * n_const
    model = workloads.random_net(ext, [6, 5], seed=seed)
    model["x_shift"] = model["x_shift"] + np.linspace(0.3, 0.7, len(ext))
    model["x_scale"] = model["x_scale"] * np.linspace(1.3, 0.6, len(ext))
    return model


def test_device_features_appended_after_parameters_and_scaled():
    """z' = [z, f_dev] (P:281 device feature; S:72 columns appended after
    the tuning parameters) for the scalar-GFLOPS and the one-hot encodings (G3):
    oracle.mlp.predict on a model with constant features f equals the brute-force
    F-input net on the space extended by one single-value list [f_c] per feature."""
    vl = [[100, 1000], [32, 384], [200, 700, 900], [64, 128]]
    for feats in ([4700.0], [0.0, 1.0, 0.0], [1.0, 0.0, 0.0]):
        model = _combined_net(vl, len(feats), seed=11 + len(feats))
        ext = vl + [[f] for f in feats]
        ref = np.array(pins.brute_times(model, ext))
        m = workloads.with_device(model, feats)
        t = sweep.times(m, vl, 0, int(np.prod([len(v) for v in vl])))
        assert np.max(np.abs(t - ref)) < 1e-12
        # the same feature values placed BEFORE the parameters (the plausible
        # mistake) give a different surface
        pre = np.array(pins.brute_times(model, [[f] for f in feats] + vl)) if len(feats) == 1 else None
        if pre is not None:
            assert np.max(np.abs(pre - ref)) > 1e-3
    # a feature left unscaled changes t as well (scale != 1, shift != 0 above)
    model = _combined_net(vl, 1, seed=3)
    unscaled = dict(model)
    unscaled["x_shift"] = model["x_shift"].copy()
    unscaled["x_scale"] = model["x_scale"].copy()
    unscaled["x_shift"][-1], unscaled["x_scale"][-1] = 0.0, 1.0
    a = sweep.times(workloads.with_device(model, [0.5]), vl, 0, 24)
    b = np.array(pins.brute_times(unscaled, vl + [[0.5]]))
    assert np.max(np.abs(a - b)) > 1e-3
