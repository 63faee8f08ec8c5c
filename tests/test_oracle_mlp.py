"""Pins for oracle.scaler and oracle.mlp."""

import warnings

import numpy as np
import pytest

from oracle import cost, mlp, scaler, space


# ---------------------------------------------------------------- scaler
def test_scaler_hand_case():
    m, s = scaler.fit_standard(np.array([[1.0], [3.0]]))
    assert m[0] == 2.0 and s[0] == 1.0
    assert np.array_equal(scaler.transform([[1.0], [3.0]], m, s), [[-1.0], [1.0]])


def test_scaler_constant_column_and_roundtrip():
    X = np.array([[5.0, 1.0], [5.0, 2.0], [5.0, 7.0]])
    m, s = scaler.fit_standard(X)
    Z = scaler.transform(X, m, s)
    assert np.all(Z[:, 0] == 0.0)
    Xr = scaler.inverse(Z, m, s)
    assert np.max(np.abs(Xr - X)) <= 1e-12


def test_scaler_matches_sklearn_standard_scaler():
    from sklearn.preprocessing import MinMaxScaler, StandardScaler
    X = np.random.default_rng(0).normal(3.0, 2.0, (500, 6))
    X[:, 2] = 4.0
    m, s = scaler.fit_standard(X)
    ref = StandardScaler().fit(X)
    assert np.allclose(m, ref.mean_, rtol=0, atol=1e-12)
    assert np.allclose(s, ref.scale_, rtol=1e-12)
    lo, rg = scaler.fit_minmax(X)
    mm = MinMaxScaler().fit(X)
    assert np.allclose(scaler.transform(X, lo, rg), mm.transform(X), atol=1e-12)


# ---------------------------------------------------------------- forward
def test_forward_zero_net():
    W, b = [np.zeros((3, 4)), np.zeros((4, 1))], [np.zeros(4), np.zeros(1)]
    assert np.all(mlp.forward(W, b, np.random.default_rng(0).normal(size=(5, 3))) == 0.0)


def test_forward_affine_1_1():
    # single layer 1->1, w=2, b=1, x=3 -> 7
    assert mlp.forward([np.array([[2.0]])], [np.array([1.0])], np.array([[3.0]]))[0] == 7.0


def test_forward_relu_1_2_1():
    # w1=[1,-1], b1=0, w2=[1,1]^T, b2=0, x=3 -> ReLU(3)+ReLU(-3) = 3
    W = [np.array([[1.0, -1.0]]), np.array([[1.0], [1.0]])]
    b = [np.zeros(2), np.zeros(1)]
    assert mlp.forward(W, b, np.array([[3.0]]))[0] == 3.0


def test_forward_hand_14_2_1():
    # W1 rows are unit vectors: hidden 0 reads z_0 - z_13, hidden 1 reads z_5;
    # by hand: h0 = max(0, 0.5 - (-1.5) + 0.25) = 2.25, h1 = max(0, -3 + 1) = 0,
    # yhat = 2 * 2.25 - 1 * 0 + 0.5 = 5.0
    W1 = np.zeros((14, 2))
    W1[0, 0], W1[13, 0], W1[5, 1] = 1.0, -1.0, 1.0
    W2 = np.array([[2.0], [-1.0]])
    z = np.zeros((1, 14))
    z[0, 0], z[0, 13], z[0, 5] = 0.5, -1.5, -3.0
    y = mlp.forward([W1, W2], [np.array([0.25, 1.0]), np.array([0.5])], z)
    assert y[0] == 5.0


# ---------------------------------------------------------------- loss/gradient
def test_loss_hand_cases():
    W, b = [np.zeros((1, 1))], [np.zeros(1)]
    # predictions [0, 0] vs targets [1, 1]: MSE = 1, sklearn form 1/2 MSE (G8)
    loss, _, _ = mlp.loss_and_grads(W, b, np.ones((2, 1)), np.ones(2), alpha=0.0)
    assert loss == 0.5
    # zero weights: L2 penalty term vanishes
    loss2, _, _ = mlp.loss_and_grads(W, b, np.ones((2, 1)), np.ones(2), alpha=1e-4)
    assert loss2 == 0.5


def test_gradient_hand_case():
    # 1->1, w=1, b=0, x=2, y=0: d/dw 1/2 (wx - y)^2 = (wx - y) x = 4
    # (SPEC S:187 quotes 8 for the un-halved MSE; G8 reading halves it)
    _, gW, gb = mlp.loss_and_grads([np.array([[1.0]])], [np.array([0.0])],
                                   np.array([[2.0]]), np.array([0.0]), alpha=0.0)
    assert gW[0][0, 0] == 4.0 and gb[0][0] == 2.0


@pytest.mark.parametrize("widths", [[2, 8, 1], [14, 16, 16, 1], [5, 7, 6, 3, 1], [3, 1], [14, 9, 1]])
def test_gradient_finite_differences(widths):
    rng = np.random.default_rng(sum(widths))
    W, b = mlp.init_glorot(widths, rng)
    X = rng.normal(size=(13, widths[0]))
    y = rng.normal(size=13)
    _, gW, gb = mlp.loss_and_grads(W, b, X, y, alpha=1e-3)
    h = 1e-6
    for P, G in list(zip(W, gW)) + list(zip(b, gb)):
        flat = P.reshape(-1)
        gflat = G.reshape(-1)
        for i in rng.choice(flat.size, size=min(flat.size, 12), replace=False):
            old = flat[i]
            flat[i] = old + h
            lp, _, _ = mlp.loss_and_grads(W, b, X, y, 1e-3)
            flat[i] = old - h
            lm, _, _ = mlp.loss_and_grads(W, b, X, y, 1e-3)
            flat[i] = old
            fd = (lp - lm) / (2 * h)
            assert abs(fd - gflat[i]) <= 1e-5 * max(1.0, abs(fd))


# ---------------------------------------------------------------- Adam
def test_adam_single_step_hand_case(golden):
    hp = golden["hyperparameters"]["value"]
    opt = mlp.Adam(hp["lr0"], hp["beta1"], hp["beta2"], hp["eps"])
    theta = np.zeros(1)
    opt.step([theta], [np.ones(1)])
    # m = 0.05, v = 0.1, lr_t = 0.0009 sqrt(0.1)/0.05, step = lr_t * 0.05/(sqrt(0.1)+eps)
    exact = -0.0009 * np.sqrt(0.1) / (np.sqrt(0.1) + 1e-9)
    assert abs(theta[0] - exact) < 1e-18
    assert abs(theta[0] - (-0.0009)) < 3e-12            # S:197 "theta ~ -0.0009"
    assert mlp.HYPER["alpha"] == hp["alpha"] and mlp.HYPER["batch_size"] == hp["batch_size"]
    assert mlp.HYPER["max_epochs"] == hp["max_epochs"] and mlp.HYPER["tol"] == hp["tol"]


def test_adam_zero_gradient_identity():
    opt = mlp.Adam(0.0009, 0.95, 0.90, 1e-9)
    theta = np.array([0.3, -1.0])
    opt.step([theta], [np.zeros(2)])
    assert np.array_equal(theta, [0.3, -1.0])


def test_one_epoch_matches_sklearn_mlpregressor():
    # the paper trains with scikit-learn; one no-shuffle epoch from the same
    # initial weights must give scikit-learn's weights and loss
    from sklearn.neural_network import MLPRegressor
    rng = np.random.default_rng(0)
    X = rng.normal(size=(450, 14))
    y = rng.normal(size=450)
    widths = [14, 12, 9, 1]
    W, b = mlp.init_glorot(widths, np.random.default_rng(1))
    reg = MLPRegressor(hidden_layer_sizes=(12, 9), solver="adam", alpha=1e-4, beta_1=0.95,
                       beta_2=0.90, learning_rate_init=0.0009, epsilon=1e-9, batch_size=200,
                       shuffle=False, max_iter=1, tol=1e-6)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        reg.partial_fit(X, y)
    for l in range(3):
        reg.coefs_[l][...] = W[l]
        reg.intercepts_[l][...] = b[l]
    del reg._optimizer
    reg.partial_fit(X, y)
    hist, _, _ = mlp.run_epochs(W, b, X, y, None, shuffle=False, max_epochs=1)
    for l in range(3):
        assert np.max(np.abs(reg.coefs_[l] - W[l])) < 1e-13
        assert np.max(np.abs(reg.intercepts_[l] - b[l])) < 1e-13
    assert abs(hist[0] - reg.loss_) < 1e-13


def test_stopping_rule_counts_stagnant_epochs():
    # all-zero data: loss stays 0 -> no improvement by tol -> stop after 11 epochs (G6)
    W, b = mlp.init_glorot([2, 3, 1], np.random.default_rng(0))
    for w in W:
        w[...] = 0.0
    for v in b:
        v[...] = 0.0
    hist, reason, _ = mlp.run_epochs(W, b, np.zeros((10, 2)), np.zeros(10),
                                     np.random.default_rng(0))
    assert reason == "tol_converged" and len(hist) == 12


# ---------------------------------------------------------------- R^2
def test_r2_cases(golden):
    ex = golden["r2_definition_example"]["value"]
    assert mlp.r2(ex["actual"], ex["predicted"]) == ex["r2"]
    assert mlp.r2([1, 2, 3], [1, 2, 3]) == 1.0
    assert mlp.r2([1, 2, 3], [2, 2, 2]) == 0.0
    assert mlp.r2([5, 5], [1, 2]) == 0.0


def test_r2_matches_sklearn():
    from sklearn.metrics import r2_score
    rng = np.random.default_rng(4)
    a, p = rng.normal(size=50), rng.normal(size=50)
    assert abs(mlp.r2(a, p) - r2_score(a, p)) < 1e-12


# ---------------------------------------------------------------- acceptance
@pytest.mark.slow
def test_training_reaches_r2_on_synthetic_surface():
    vl = [[64, 128, 256, 512, 1024], [32, 64, 128]] * 7
    r = [len(v) for v in vl]
    idx = space.sample_indices(r, 10000, np.random.default_rng(1))
    cm = cost.make_cost_model(vl, seed=1, noise_sigma=0.0)
    X = space.values_of(space.decode(idx, r), vl)
    y = cm.cost(idx)
    tr, te = space.split(10000, 0.75, np.random.default_rng(2))
    model, _ = mlp.train(X[tr], y[tr], [64, 64], seed=3, max_epochs=60)
    assert mlp.r2(y[te], mlp.predict(model, X[te])) >= 0.90


def test_predict_row_purity_and_ensemble_mean():
    rng = np.random.default_rng(9)
    X = rng.normal(size=(40, 3))
    y = X @ np.array([1.0, -2.0, 0.5]) + 3.0
    model, _ = mlp.train(X, y, [8], seed=1, ensemble=2, max_epochs=5)
    t = mlp.predict(model, X)
    perm = rng.permutation(40)
    assert np.array_equal(mlp.predict(model, X[perm]), t[perm])
    one = [dict(model, members=[m]) for m in model["members"]]
    assert np.allclose(t, (mlp.predict(one[0], X) + mlp.predict(one[1], X)) / 2, rtol=0, atol=1e-15)


def test_run_epochs_given_orders_equal_drawn_orders():
    # passing the epoch orders as an input (the GPU-training parity path) is the
    # same computation as drawing them from the rng inside the loop
    rng = np.random.default_rng(42)
    X = rng.standard_normal((450, 5))
    y = rng.standard_normal(450)
    W0, b0 = mlp.init_glorot([5, 8, 8, 1], np.random.default_rng(1))
    r1 = np.random.default_rng(9)
    W1, b1 = [w.copy() for w in W0], [v.copy() for v in b0]
    h1, _, _ = mlp.run_epochs(W1, b1, X, y, r1, max_epochs=4)
    r2 = np.random.default_rng(9)
    perms = [r2.permutation(450) for _ in range(4)]
    W2, b2 = [w.copy() for w in W0], [v.copy() for v in b0]
    h2, _, _ = mlp.run_epochs(W2, b2, X, y, None, max_epochs=4, perms=perms)
    assert h1 == h2
    assert all(np.array_equal(a, c) for a, c in zip(W1 + b1, W2 + b2))
