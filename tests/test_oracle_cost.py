"""Pins for oracle.cost (the synthetic solver-time surface)."""

import itertools
import math

import numpy as np

from oracle import cost, space


def _vl():
    return [[100, 200, 400, 800], [32, 64, 128], [100, 300, 1000], [32, 96, 384]]


def test_calibrated_window_exact(golden):
    lo, hi = golden["time_window_s"]["value"]
    vl = _vl()
    cm = cost.make_cost_model(vl, seed=4, noise_sigma=0.0)
    n = space.cardinality([len(v) for v in vl])
    t = cm.cost(np.arange(n, dtype=np.uint64))
    assert abs(t.min() - lo) < 1e-12 and abs(t.max() - hi) < 1e-12


def test_optimum_on_grid_gives_base():
    vl = _vl()
    opt = [200, 64, 300, 96]
    cm = cost.make_cost_model(vl, seed=9, noise_sigma=0.0, optima=opt)
    d = [vl[j].index(opt[j]) for j in range(4)]
    i = space.encode(d, [len(v) for v in vl])
    assert abs(cm.cost(np.array([i]))[0] - cost.T_LO) < 1e-15


def test_argmin_is_nearest_log2_grid_point():
    # with c_int = 0 the surface is separable: the optimum is the per-axis nearest
    # grid point in log2 distance, checked by full enumeration
    vl = _vl()
    for seed in range(5):
        cm = cost.make_cost_model(vl, seed=seed, noise_sigma=0.0, c_int_scale=0.0)
        r = [len(v) for v in vl]
        t = cm.cost(np.arange(space.cardinality(r), dtype=np.uint64))
        best = space.decode(int(np.argmin(t)), r)
        opts = [cm.g_opt[0], cm.v_opt[0], cm.g_opt[1], cm.v_opt[1]]
        for j in range(4):
            dist = [abs(math.log2(x / opts[j])) for x in vl[j]]
            assert best[j] == int(np.argmin(dist))


def test_noise_deterministic_and_gaussian():
    vl = _vl()
    cm = cost.make_cost_model(vl, seed=2, noise_sigma=0.02)
    idx = np.arange(space.cardinality([len(v) for v in vl]), dtype=np.uint64)
    a = cm.noise(idx)
    assert np.array_equal(a, cm.noise(idx))
    big = cm.noise(np.arange(200000, dtype=np.uint64))
    assert abs(big.mean()) < 3 * 0.02 / math.sqrt(200000)
    assert abs(big.std() - 0.02) < 0.0005


def test_quadratic_form_hand_value():
    # one kernel, hand arithmetic of A x^2 + B y^2 + c x y at x = 1, y = -2
    vl = [[1, 2, 4], [1, 2, 4]]
    cm = cost.make_cost_model(vl, seed=1, noise_sigma=0.0, optima=[1, 4])
    A, B, c = cm.A[0], cm.B[0], cm.c_int
    q = cm.q(np.array([[2.0, 1.0]]))[0]
    assert abs(q - (A * 1 + B * 4 + c * (1 * -2))) < 1e-12
    # enumeration of all 9 points for the calibration extrema
    qs = [cm.q(np.array([[g, v]], float))[0] for g, v in itertools.product([1, 2, 4], [1, 2, 4])]
    assert abs(min(qs) - cm.q_min) < 1e-12 and abs(max(qs) - cm.q_max) < 1e-12
