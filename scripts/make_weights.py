#!/usr/bin/env python3
"""Train the BASELINE-config surrogates with the ORACLE and write weights/*.npz.

Calls only oracle/ (and workloads/ for value lists and file I/O), so every
weight file is an oracle product, never a CUDA one (task rule ③).  The paper's
workflow: sample configs at random, label them
(here: the synthetic surface, oracle/cost.py, standing in for SENSEI timings),
split 75/25, fit StandardScaler on the training split, train the FCNN with the
Table "Hyperparameter" values, report R^2 on both splits.

    python scripts/make_weights.py [cfg1 cfg2 cfg3 cfg4 cfg5]
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
import workloads  # noqa: E402

MASTER_SEED = 0x2306014011


def dataset(value_lists, n, device, seed):
    radices = [len(v) for v in value_lists]
    rng = np.random.default_rng([seed, 0x5A3B])
    idx = oracle.space.sample_indices(radices, n, rng)
    cm = oracle.cost.make_cost_model(value_lists, seed=seed, device=device, noise_sigma=0.02)
    X = oracle.space.values_of(oracle.space.decode(idx, radices), value_lists)
    y = cm.cost(idx)
    return X, y


def train_single(wl, seed):
    vl = workloads.space(wl.space)
    n = wl.train_n
    X, y = dataset(vl, n, "P100", seed)
    tr, te = oracle.space.split(n, 0.75, np.random.default_rng([seed, 0x5B11]))
    model, reps = oracle.mlp.train(X[tr], y[tr], wl.hidden, seed=seed, ensemble=wl.ensemble)
    r2_tr = oracle.mlp.r2(y[tr], oracle.mlp.predict(model, X[tr]))
    r2_te = oracle.mlp.r2(y[te], oracle.mlp.predict(model, X[te]))
    return model, reps, r2_tr, r2_te


def train_combined(wl, seed):
    """Combined training: one dataset per device, device feature
    appended (G3), 75/25 split per device, pooled -> 22,500 training rows."""
    vl = workloads.space(wl.space)
    Xs, ys, Xt, yt = [], [], [], []
    for d, dev in enumerate(wl.devices):
        X, y = dataset(vl, 10000, dev, seed + d)
        f = np.asarray(workloads.device_features(wl.device_encoding, dev))
        X = np.concatenate([X, np.broadcast_to(f, (X.shape[0], f.size))], axis=1)
        tr, te = oracle.space.split(X.shape[0], 0.75, np.random.default_rng([seed, d, 0x5B11]))
        Xs.append(X[tr]); ys.append(y[tr]); Xt.append(X[te]); yt.append(y[te])
    Xtr, ytr = np.concatenate(Xs), np.concatenate(ys)
    Xte, yte = np.concatenate(Xt), np.concatenate(yt)
    model, reps = oracle.mlp.train(Xtr, ytr, wl.hidden, seed=seed, ensemble=wl.ensemble)
    r2_tr = oracle.mlp.r2(ytr, oracle.mlp.predict(model, Xtr))
    r2_te = oracle.mlp.r2(yte, oracle.mlp.predict(model, Xte))
    return model, reps, r2_tr, r2_te


def main(names):
    for name in names:
        wl = workloads.WORKLOADS[name]
        seed = MASTER_SEED + sum(map(ord, name))
        t0 = time.time()
        if wl.device_encoding:
            model, reps, r2_tr, r2_te = train_combined(wl, seed)
        else:
            model, reps, r2_tr, r2_te = train_single(wl, seed)
        meta = dict(r2_train=r2_tr, r2_test=r2_te, epochs=[r["epochs"] for r in reps],
                    stop=[r["stop_reason"] for r in reps], seed=seed,
                    final_loss=[r["loss_history"][-1] for r in reps])
        workloads.save_model(model, wl.weights, meta={"json": json.dumps(meta)})
        print(name, wl.weights, f"{time.time() - t0:.1f}s", json.dumps(meta))


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg1", "cfg2", "cfg5", "cfg3", "cfg4"])
