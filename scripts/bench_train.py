#!/usr/bin/env python3
"""GPU training vs the float64 oracle on the paper's training problem
(SURVEY 8(f) NEXT-4): 10,000 samples, 75/25 split -> 7,500 training rows
(P:307), 14-128-128-1, batch 200, up to 200 epochs, the paper's Adam
hyperparameters.  Prints one JSON line.

    python scripts/bench_train.py [--H 128] [--n 7500] [--epochs 200] [--oracle-epochs 5]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_14011_b200 as pk  # noqa: E402
import workloads  # noqa: E402
from oracle import mlp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--H", type=int, default=128)
    ap.add_argument("--n", type=int, default=7500)
    ap.add_argument("--epochs", type=int, default=200)
    ap.add_argument("--oracle-epochs", type=int, default=5)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ensemble", type=int, default=1, help="members trained at once (cfg 4: 8)")
    a = ap.parse_args()
    vl = workloads.space("cfg2")
    X, y = workloads.training_rows(vl, a.n + 2500, seed=5)
    Xt, yt = X[a.n:], y[a.n:]
    X, y = X[:a.n], y[:a.n]
    W0, b0 = workloads.glorot_init([14, a.H, a.H, 1], seed=5)
    perms = workloads.epoch_permutations(a.n, a.epochs, seed=6)
    hyper = dict(pk.TRAIN_HYPER, max_epochs=a.epochs)
    pk.train(W0, b0, X[:400], y[:400], None, dict(hyper, max_epochs=1))  # warm-up (module load, first launch)
    E = a.ensemble
    members = [(W0, b0)] + [workloads.glorot_init([14, a.H, a.H, 1], seed=5 + e) for e in range(1, E)]
    eperms = np.stack([perms] + [workloads.epoch_permutations(a.n, a.epochs, seed=6 + e) for e in range(1, E)])
    times = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        res = pk.train_ensemble(members, X, y, eperms, hyper)
        times.append(time.perf_counter() - t0)
    gpu_s = min(times)
    W, b, hist, reason = res[0]
    steps = sum(len(r[2]) for r in res) * -(-a.n // hyper["batch_size"])
    # oracle (float64 numpy) on the first epochs of the same fit, per step
    Wo, bo = [w.copy() for w in W0], [v.copy() for v in b0]
    t0 = time.perf_counter()
    mlp.run_epochs(Wo, bo, X, y, None, hyper=dict(hyper, max_epochs=a.oracle_epochs), perms=perms)
    or_s = time.perf_counter() - t0
    or_steps = a.oracle_epochs * -(-a.n // hyper["batch_size"])
    flops_step = 2 * 3 * hyper["batch_size"] * (14 * a.H + a.H * a.H + a.H)  # forward + 2x backward MACs
    out = {"metric": "FCNN training steps/sec (batch 200, Adam)", "value": steps / gpu_s, "unit": "steps/s",
           "ms_per_step": gpu_s / steps * 1e3, "fit_s": gpu_s, "epochs": len(hist), "stop": reason,
           "samples_per_s": steps * hyper["batch_size"] / gpu_s,
           "achieved_gflops": flops_step * steps / gpu_s / 1e9,
           "r2_test": mlp.r2(yt, mlp.forward(W, b, Xt)), "final_loss": hist[-1],
           "config": {"net": f"14-{a.H}-{a.H}-1" + (f" x{E}" if E > 1 else ""), "n_train": a.n,
                      "batch": hyper["batch_size"], "dtype": "f32",
                      "launch": f"1 launch: {E} cluster(s) of {a.H // 16} CTAs for the whole fit"},
           "cpu_baseline": {"value": or_steps / or_s, "unit": "steps/s", "kind": "oracle",
                            "cores": os.cpu_count(), "sample": f"first {a.oracle_epochs} epochs, numpy float64"}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
