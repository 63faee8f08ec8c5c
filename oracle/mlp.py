"""Fully connected ReLU regression network (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

The paper's surrogate: input = tuning parameters, hidden layers
"activated by the rectified linear unit", identity output = solver runtime;
fitted with scikit-learn using Adam and Table "Hyperparameter for the
artificial neural network":

    alpha = 1e-4, beta1 = 0.95, beta2 = 0.90, lr0 = 0.0009, max epochs 200,
    batch 200, tol 1e-6, eps 1e-9.

Because the paper names scikit-learn's MLPRegressor defaults for the rest,
this module restates that algorithm, in its order:
Glorot-uniform init of weights and biases, loss = 1/2 mean squared error +
alpha/(2B) sum ||W||_F^2 (biases excluded), output delta = yhat - y,
dW = (A^T delta + alpha W)/B, db = mean(delta), ReLU subgradient 0 at 0, Adam
with lr_t = lr0 sqrt(1-beta2^t)/(1-beta1^t), epoch loss = sample-weighted mean
of batch losses, stop after more than 10 epochs without improving by tol (G6).
Targets are standardised as well (reading G4).

Weights are stored row-major fan_in x fan_out.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import scaler as _scaler

HYPER = dict(alpha=1e-4, beta1=0.95, beta2=0.90, lr0=0.0009, max_epochs=200,
             batch_size=200, tol=1e-6, eps=1e-9, n_iter_no_change=10)


def init_glorot(widths, rng: np.random.Generator):
    """Glorot-uniform U(+-sqrt(6/(fan_in+fan_out))) for W and b (sklearn _init_coef)."""
    W, b = [], []
    for fan_in, fan_out in zip(widths[:-1], widths[1:]):
        bound = np.sqrt(6.0 / (fan_in + fan_out))
        W.append(rng.uniform(-bound, bound, (fan_in, fan_out)))
        b.append(rng.uniform(-bound, bound, fan_out))
    return W, b


def forward_layers(W, b, X):
    """All activations [X, h_1, ..., h_{L-1}, yhat]: h_l = max(0, h_{l-1} W_l + b_l)
    for hidden layers, identity on the output (P:54 forward propagation)."""
    acts = [np.asarray(X, dtype=np.float64)]
    L = len(W)
    for l in range(L):
        z = acts[-1] @ W[l] + b[l]
        if l < L - 1:
            z = np.maximum(z, 0.0)
        acts.append(z)
    return acts


def forward(W, b, X) -> np.ndarray:
    """Network output (standardised units), shape (n,)."""
    return forward_layers(W, b, X)[-1][:, 0]


def loss_and_grads(W, b, X, y, alpha: float):
    """sklearn-form loss and its exact gradient by backpropagation (P:54 chain rule)."""
    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64).reshape(-1, 1)
    n = X.shape[0]
    if n == 0:
        raise ValueError("empty batch")
    acts = forward_layers(W, b, X)
    loss = ((y - acts[-1]) ** 2).mean() / 2.0
    loss += 0.5 * alpha * sum(float(np.dot(w.ravel(), w.ravel())) for w in W) / n
    L = len(W)
    gW = [None] * L
    gb = [None] * L
    delta = acts[-1] - y
    for l in range(L - 1, -1, -1):
        gW[l] = (acts[l].T @ delta + alpha * W[l]) / n
        gb[l] = delta.mean(axis=0)
        if l > 0:
            delta = delta @ W[l].T
            delta[acts[l] == 0] = 0.0  # ReLU subgradient 0 where the unit is off
    return loss, gW, gb


@dataclass
class Adam:
    """Adam in the sklearn form ("adaptive moment estimation")."""

    lr0: float
    beta1: float
    beta2: float
    eps: float
    t: int = 0
    m: list = field(default_factory=list)
    v: list = field(default_factory=list)

    def step(self, params, grads):
        if not self.m:
            self.m = [np.zeros_like(p) for p in params]
            self.v = [np.zeros_like(p) for p in params]
        self.t += 1
        self.m = [self.beta1 * m + (1 - self.beta1) * g for m, g in zip(self.m, grads)]
        self.v = [self.beta2 * v + (1 - self.beta2) * g * g for v, g in zip(self.v, grads)]
        lr_t = self.lr0 * np.sqrt(1 - self.beta2 ** self.t) / (1 - self.beta1 ** self.t)
        for p, m, v in zip(params, self.m, self.v):
            p += -lr_t * m / (np.sqrt(v) + self.eps)
        return lr_t


def run_epochs(W, b, Xs, ys, rng, hyper=None, shuffle=True, max_epochs=None, opt=None, perms=None):
    """The minibatch epoch loop on already-standardised data; mutates W, b.
    perms: optional [epochs, n] epoch orders given as an input (the random
    numbers of the shuffle passed in, so another implementation can be run on
    the same orders); otherwise each epoch draws rng.permutation(n).

    Returns (loss_history, stop_reason, opt)."""
    h = dict(HYPER)
    if hyper:
        h.update(hyper)
    n = Xs.shape[0]
    bs = min(h["batch_size"], n)
    if opt is None:
        opt = Adam(h["lr0"], h["beta1"], h["beta2"], h["eps"])
    params = list(W) + list(b)
    history = []
    best = np.inf
    no_improve = 0
    reason = "max_epochs"
    idx = np.arange(n)
    for ep in range(max_epochs if max_epochs is not None else h["max_epochs"]):
        if perms is not None:
            idx = np.asarray(perms[ep], dtype=np.int64)
        elif shuffle:
            idx = rng.permutation(n)
        acc = 0.0
        for s in range(0, n, bs):
            bi = idx[s:s + bs]
            loss, gW, gb = loss_and_grads(W, b, Xs[bi], ys[bi], h["alpha"])
            acc += loss * len(bi)
            opt.step(params, list(gW) + list(gb))
        history.append(acc / n)
        if history[-1] > best - h["tol"]:
            no_improve += 1
        else:
            no_improve = 0
        if history[-1] < best:
            best = history[-1]
        if no_improve > h["n_iter_no_change"]:
            reason = "tol_converged"
            break
    return history, reason, opt


def r2(actual, predicted) -> float:
    """Eq. (R_square): 1 - sum (y - yhat)^2 / sum (y - ybar)^2; a zero
    denominator returns 0."""
    a = np.asarray(actual, dtype=np.float64)
    p = np.asarray(predicted, dtype=np.float64)
    if a.shape != p.shape or a.size == 0:
        raise ValueError("equal non-zero lengths required")
    den = float(((a - a.mean()) ** 2).sum())
    if den == 0.0:
        return 0.0
    return 1.0 - float(((a - p) ** 2).sum()) / den


def make_model(widths, members, x_shift, x_scale, y_mean, y_scale,
               const_features=None, x_scaler="standard"):
    """The model record both sides consume (see workloads/__init__.py)."""
    return dict(widths=[int(w) for w in widths],
                members=[dict(W=[np.asarray(w, np.float64) for w in m["W"]],
                              b=[np.asarray(v, np.float64) for v in m["b"]]) for m in members],
                x_shift=np.asarray(x_shift, np.float64), x_scale=np.asarray(x_scale, np.float64),
                y_mean=float(y_mean), y_scale=float(y_scale),
                const_features=(np.zeros(0) if const_features is None
                                else np.asarray(const_features, np.float64)),
                x_scaler=x_scaler)


def train(X_train, y_train, hidden, seed: int, ensemble: int = 1, hyper=None,
          x_scaler="standard", max_epochs=None):
    """Fit the scalers on the training split, then E independently initialised
    members on the same data (G15); returns (model, report)."""
    X_train = np.asarray(X_train, np.float64)
    y_train = np.asarray(y_train, np.float64)
    fit = _scaler.fit_standard if x_scaler == "standard" else _scaler.fit_minmax
    xs, xsc = fit(X_train)
    ym, ysc = _scaler.fit_standard(y_train.reshape(-1, 1))
    Xs = _scaler.transform(X_train, xs, xsc)
    ys = (y_train - ym[0]) / ysc[0]
    widths = [X_train.shape[1]] + list(hidden) + [1]
    members, reports = [], []
    for e in range(ensemble):
        rng = np.random.default_rng([seed, e, 0x1417])
        W, b = init_glorot(widths, rng)
        hist, reason, _ = run_epochs(W, b, Xs, ys, rng, hyper=hyper, max_epochs=max_epochs)
        members.append(dict(W=W, b=b))
        reports.append(dict(loss_history=hist, stop_reason=reason, epochs=len(hist)))
    model = make_model(widths, members, xs, xsc, ym[0], ysc[0], x_scaler=x_scaler)
    return model, reports


def predict(model, X) -> np.ndarray:
    """t = (1/E) sum_e (mu_y + sigma_y * yhat_e(z)), z = (x - shift)/scale (S:208-216,
    SURVEY c1).  X holds raw values; constant device features (if any) are
    appended after the tuning parameters."""
    X = np.asarray(X, np.float64)
    cf = model["const_features"]
    if cf.size:
        X = np.concatenate([X, np.broadcast_to(cf, (X.shape[0], cf.size))], axis=1)
    Z = _scaler.transform(X, model["x_shift"], model["x_scale"])
    t = np.zeros(X.shape[0])
    for m in model["members"]:
        t += model["y_mean"] + model["y_scale"] * forward(m["W"], m["b"], Z)
    return t / len(model["members"])
