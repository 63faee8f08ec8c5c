"""GPU-side training against the float64 oracle
(oracle/mlp.py run_epochs) on the same seeded inputs: initial weights, data and
epoch orders from workloads (nothing shared but the inputs).

Tolerances: the trainer is FP32, the oracle float64.
Adam's first steps are ~lr0 sign(g) per parameter, so a few steps agree to
FP32 rounding; over a full fit the two trajectories drift apart the way any
FP32 and float64 runs of the same minibatch sequence do, so the full-fit test
compares what the fit is for: the loss curve, the stopping epoch and the
predictions of the trained nets."""

import numpy as np
import pytest

import workloads
from oracle import mlp
from tests.helpers import need_gpu

pytestmark = pytest.mark.gpu

HYPER = dict(alpha=1e-4, beta1=0.95, beta2=0.90, lr0=0.0009, eps=1e-9, tol=1e-6, batch_size=200,
             n_iter_no_change=10)


def _oracle(W, b, X, y, perms, epochs):
    W = [w.copy() for w in W]
    b = [v.copy() for v in b]
    h = dict(HYPER, max_epochs=epochs)
    hist, reason, _ = mlp.run_epochs(W, b, X, y, None, hyper=h, perms=perms)
    return W, b, hist, reason


@pytest.mark.parametrize("H,n,epochs", [(32, 1000, 1), (128, 600, 2), (64, 437, 3)])
def test_train_first_steps_match_oracle(H, n, epochs):
    pk = need_gpu()
    vl = workloads.space("cfg2")
    X, y = workloads.training_rows(vl, n, seed=H + n)
    W0, b0 = workloads.glorot_init([14, H, H, 1], seed=H)
    perms = workloads.epoch_permutations(n, epochs, seed=n)
    Wg, bg, hg, _ = pk.train(W0, b0, X, y, perms, dict(HYPER, max_epochs=epochs))
    Wo, bo, ho, _ = _oracle(W0, b0, X, y, perms, epochs)
    assert len(hg) == len(ho) == epochs
    assert np.allclose(hg, ho, rtol=1e-5, atol=0.0), (hg, ho)
    steps = epochs * -(-n // 200)
    for a, c, p0 in zip(Wg + bg, Wo + bo, W0 + b0):
        moved = np.abs(c - p0)  # each step moves a parameter by <= ~lr0 * 3.2 (|m| / sqrt(v) bound)
        assert moved.max() <= steps * 0.0009 * 3.2
        # FP32 vs float64 on the same steps: rounding of p (|p| 2^-24 per step) plus
        # the update's relative rounding; a sign flip of a ~0 gradient costs 2 lr0
        err = np.abs(a - c)
        bad = err > 1e-5 * steps * 0.0009 + 4e-7 * np.abs(c)
        assert bad.mean() <= 0.002, f"{bad.sum()} of {bad.size} parameters off (max {err.max():.3e})"


def test_train_full_fit_matches_oracle():
    # cfg1-sized fit (14-32-32-1, paper hyperparameters, up to 200 epochs)
    pk = need_gpu()
    vl = workloads.space("cfg2")
    n = 1600
    X, y = workloads.training_rows(vl, n + 400, seed=7)
    Xt, yt = X[n:], y[n:]
    X, y = X[:n], y[:n]
    W0, b0 = workloads.glorot_init([14, 32, 32, 1], seed=3)
    perms = workloads.epoch_permutations(n, 200, seed=11)
    Wg, bg, hg, rg = pk.train(W0, b0, X, y, perms, dict(HYPER, max_epochs=200))
    Wo, bo, ho, ro = _oracle(W0, b0, X, y, perms, 200)
    m = min(len(hg), len(ho))
    rel = np.abs(np.array(hg[:m]) - np.array(ho[:m])) / np.array(ho[:m])
    assert rel.max() <= 2e-2, rel.max()
    assert abs(len(hg) - len(ho)) <= 15 and rg == ro, (len(hg), rg, len(ho), ro)
    pg = mlp.forward(Wg, bg, Xt)
    po = mlp.forward(Wo, bo, Xt)
    assert abs(mlp.r2(yt, pg) - mlp.r2(yt, po)) <= 0.01
    # an FP32 emulation of the same fit differs from float64 by 0.095 at most here
    assert np.abs(pg - po).max() <= 0.25  # standardised units
    assert mlp.r2(yt, pg) >= 0.9


def test_train_rejects_bad_input():
    pk = need_gpu()
    vl = workloads.space("cfg2")
    X, y = workloads.training_rows(vl, 300, seed=1)
    W0, b0 = workloads.glorot_init([14, 48, 48, 1], seed=1)
    with pytest.raises(pk.SurrogateError):
        pk.train(W0, b0, X, y)  # H = 48 is outside {32, 64, 128}
    W0, b0 = workloads.glorot_init([14, 32, 32, 1], seed=1)
    bad = workloads.epoch_permutations(300, 2, seed=1)
    bad[1, 7] = 300
    with pytest.raises(pk.SurrogateError):
        pk.train(W0, b0, X, y, bad, dict(HYPER, max_epochs=2))
    with pytest.raises(pk.SurrogateError):
        pk.train(W0, b0, X, y, None, dict(HYPER, max_epochs=2, batch_size=512))


def test_train_ensemble_members_independent_and_bitwise():
    # E clusters in one launch: each member equals its own single-member fit bitwise,
    # and member 1's first steps match the oracle on its own inputs
    pk = need_gpu()
    vl = workloads.space("cfg2")
    n, E, ep = 700, 3, 2
    X, y = workloads.training_rows(vl, n, seed=21)
    inits = [workloads.glorot_init([14, 32, 32, 1], seed=30 + e) for e in range(E)]
    perms = np.stack([workloads.epoch_permutations(n, ep, seed=40 + e) for e in range(E)])
    res = pk.train_ensemble(inits, X, y, perms, dict(HYPER, max_epochs=ep))
    for e in range(E):
        We, be, he, _ = pk.train(inits[e][0], inits[e][1], X, y, perms[e], dict(HYPER, max_epochs=ep))
        assert all(np.array_equal(a, c) for a, c in zip(res[e][0] + res[e][1], We + be))
        assert res[e][2] == he
    Wo, bo, ho, _ = _oracle(inits[1][0], inits[1][1], X, y, perms[1], ep)
    assert np.allclose(res[1][2], ho, rtol=1e-5, atol=0.0)
    err = max(np.abs(a - c).max() for a, c in zip(res[1][0] + res[1][1], Wo + bo))
    assert err <= 1e-5 * ep * 4 * 0.0009 + 4e-7 * 3
