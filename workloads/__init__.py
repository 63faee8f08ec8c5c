"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no decode, no normalisation, no
forward pass, no ranking): only the search-space value lists of the BASELINE
configs, the network shapes and k, loading of weight files written by
``scripts/make_weights.py`` (which calls only ``oracle/``), and seeded
generators of hand-built nets used as pins.

Spaces (parameter order = Table "Tuning Parameters",
P:253-266: xi-limiter gang, xi-limiter vector, eta-limiter gang, ... ,
update-solution vector; gang at even positions, vector at odd):

  cfg1 tiny    gang {100, 1000}, vector {32, 384}            2^14      = 16,384
  cfg2 paper-  gang {64..1024} x2 (r=5), vector {32,64,128}  15^7      = 170,859,375
       shaped
  cfg3 deeper  gang r=5, vector {32..256} (r=4)              20^7      = 1,280,000,000
  cfg5 large   gang {16..1024} (r=7), vector {32..256} (r=4) 28^7      = 13,492,928,512
  paper        gang 100..1000 step 100, vector 32..384 step 32  10^7 12^7 = 3.58e14
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WEIGHTS_DIR = os.path.join(ROOT, "weights")

PARAM_NAMES = [f"{k} {kind}" for k in ("xi limiter", "eta limiter", "xi flux", "eta flux",
                                        "source term", "right hand side", "update solution")
               for kind in ("gang", "vector")]


def _interleave(gang, vec, kernels=7):
    out = []
    for _ in range(kernels):
        out.append(list(gang))
        out.append(list(vec))
    return out


SPACES = {
    "tiny": _interleave([100, 1000], [32, 384]),
    "cfg2": _interleave([64, 128, 256, 512, 1024], [32, 64, 128]),
    "cfg3": _interleave([64, 128, 256, 512, 1024], [32, 64, 128, 256]),
    "cfg5": _interleave([16, 32, 64, 128, 256, 512, 1024], [32, 64, 128, 256]),
    "paper": _interleave(list(range(100, 1001, 100)), list(range(32, 385, 32))),
}

# Table "GPU specification", used as device features (G3).
DEVICES = {"C2075": 513.0, "P100": 4700.0, "V100": 7500.0}


@dataclass
class Workload:
    name: str
    space: str
    hidden: list
    k: int
    precision: str            # "fp16" | "bf16" | "tf32" | "fp32" (FP32 path: 3xFP16 / 3xTF32 + FP32 final)
    weights: str              # file stem under weights/
    train_n: int
    ensemble: int = 1
    device_encoding: str | None = None   # None | "gflops" | "onehot"
    devices: list = field(default_factory=list)
    note: str = ""
    window: int | None = None  # bench step = this many configs from |S|/3 (None: the whole space)


# BASELINE.json configs (G5 for unstated widths).
WORKLOADS = {
    "cfg1": Workload("cfg1", "tiny", [32, 32], 1, "fp32", "tiny_14-32-32-1", 1638,
                     note="tiny space, FCNN 14-32-32-1 FP32, top-1"),
    # headline precision FP16: the 16-bit tensor rate within the north star's
    # 1e-3 bound (BF16 reaches 2.6e-3 on these nets)
    "cfg2": Workload("cfg2", "cfg2", [128, 128], 16, "fp16", "cfg2_14-128-128-1", 10000,
                     note="paper-shaped space 15^7, FCNN 14-128-128-1, top-16, 1 GPU"),
    "cfg2_fp32": Workload("cfg2_fp32", "cfg2", [128, 128], 16, "fp32", "cfg2_14-128-128-1", 10000,
                          note="cfg2 on the FP32 path (3xFP16 hidden + FP32 final)"),
    "cfg2_bf16": Workload("cfg2_bf16", "cfg2", [128, 128], 16, "bf16", "cfg2_14-128-128-1", 10000,
                          note="cfg2 with BF16 hidden layers"),
    "cfg3": Workload("cfg3", "cfg3", [256, 256, 256], 64, "fp16", "cfg3_14-256-256-256-1", 10000,
                     note="deeper net 14-256-256-256-1 (16-bit hidden layers), 20^7 configs, top-64"),
    "cfg4": Workload("cfg4", "cfg2", [128, 128], 16, "fp16", "cfg4_17-128-128-1_x8", 7500,
                     ensemble=8, device_encoding="onehot", devices=["C2075", "P100", "V100"],
                     note="combined-GPU-model variant: 14 params + one-hot GPU type, 8-member ensemble"),
    "cfg5": Workload("cfg5", "cfg5", [128, 128], 1024, "fp16", "cfg5_14-128-128-1", 10000,
                     note="large sweep 28^7 = 1.35e10 configs, top-1024 per rank"),
    "paper": Workload("paper", "paper", [128, 128], 1024, "fp16", "paper_14-128-128-1", 10000, window=1 << 35,
                      note="the paper's own space, 10^7 12^7 = 3.58e14 configs (P:241), top-1024; "
                           "SURVEY 8(f) NEXT-2 (bench: a bounded index window, full-space time projected)"),
}


def space(name: str) -> list:
    return [list(v) for v in SPACES[name]]


def radices(name: str) -> list:
    return [len(v) for v in SPACES[name]]


def load_model(stem: str) -> dict:
    """Read weights/<stem>.npz into the model record:
    {widths, members: [{W: [fan_in x fan_out], b: [...]}], x_shift, x_scale,
     y_mean, y_scale, const_features, x_scaler}."""
    path = os.path.join(WEIGHTS_DIR, stem + ".npz")
    z = np.load(path, allow_pickle=False)
    widths = [int(w) for w in z["widths"]]
    E = int(z["ensemble"])
    L = len(widths) - 1
    members = [dict(W=[z[f"W_{e}_{l}"] for l in range(L)], b=[z[f"b_{e}_{l}"] for l in range(L)])
               for e in range(E)]
    return dict(widths=widths, members=members, x_shift=z["x_shift"], x_scale=z["x_scale"],
                y_mean=float(z["y_mean"]), y_scale=float(z["y_scale"]),
                const_features=z["const_features"], x_scaler=str(z["x_scaler"]))


def save_model(model: dict, stem: str, meta: dict | None = None) -> str:
    os.makedirs(WEIGHTS_DIR, exist_ok=True)
    arrays = dict(widths=np.asarray(model["widths"], np.int64),
                  ensemble=np.int64(len(model["members"])),
                  x_shift=model["x_shift"], x_scale=model["x_scale"],
                  y_mean=np.float64(model["y_mean"]), y_scale=np.float64(model["y_scale"]),
                  const_features=np.asarray(model["const_features"], np.float64),
                  x_scaler=np.str_(model.get("x_scaler", "standard")))
    for e, m in enumerate(model["members"]):
        for l, (w, b) in enumerate(zip(m["W"], m["b"])):
            arrays[f"W_{e}_{l}"] = np.asarray(w, np.float64)
            arrays[f"b_{e}_{l}"] = np.asarray(b, np.float64)
    if meta:
        for key, val in meta.items():
            arrays["meta_" + key] = np.asarray(val)
    path = os.path.join(WEIGHTS_DIR, stem + ".npz")
    np.savez(path, **arrays)
    return path


def with_device(model: dict, features) -> dict:
    """A copy of a combined-training model with its constant device features set
    (raw values appended after the 14 tuning parameters; G3)."""
    m = dict(model)
    m["const_features"] = np.asarray(features, np.float64)
    return m


def device_features(encoding: str, device: str) -> list:
    if encoding == "gflops":
        return [DEVICES[device]]
    if encoding == "onehot":
        return [1.0 if d == device else 0.0 for d in sorted(DEVICES)]
    raise ValueError(encoding)


# ---------------------------------------------------------------------------
# hand-built nets (pins); scalers chosen so that |z| <= 1 on every value list
# ---------------------------------------------------------------------------

def _unit_scaler(value_lists):
    lo = np.array([min(v) for v in value_lists], np.float64)
    hi = np.array([max(v) for v in value_lists], np.float64)
    shift = (lo + hi) / 2.0
    scale = np.where(hi > lo, (hi - lo) / 2.0, 1.0)
    return shift, scale


def random_net(value_lists, hidden, seed: int, y_mean=1.4, y_scale=0.3, ensemble=1):
    """Glorot-scaled random weights (distribution of a trained net)."""
    rng = np.random.default_rng([seed, 0x5EED])
    widths = [len(value_lists)] + list(hidden) + [1]
    members = []
    for _ in range(ensemble):
        W, b = [], []
        for fi, fo in zip(widths[:-1], widths[1:]):
            bound = np.sqrt(6.0 / (fi + fo))
            W.append(rng.uniform(-bound, bound, (fi, fo)))
            b.append(rng.uniform(-bound, bound, fo))
        members.append(dict(W=W, b=b))
    shift, scale = _unit_scaler(value_lists)
    return dict(widths=widths, members=members, x_shift=shift, x_scale=scale,
                y_mean=float(y_mean), y_scale=float(y_scale), const_features=np.zeros(0),
                x_scaler="custom")


def all_ties_net(value_lists, hidden, c=0.25, y_mean=1.0, y_scale=0.5):
    """Zero weights, output bias c: t == y_mean + y_scale * c for every config, so the
    top-k must be exactly begin..begin+k-1 (SURVEY §4 derived pin 2)."""
    widths = [len(value_lists)] + list(hidden) + [1]
    W = [np.zeros((fi, fo)) for fi, fo in zip(widths[:-1], widths[1:])]
    b = [np.zeros(fo) for fo in widths[1:]]
    b[-1][0] = c
    shift, scale = _unit_scaler(value_lists)
    return dict(widths=widths, members=[dict(W=W, b=b)], x_shift=shift, x_scale=scale,
                y_mean=float(y_mean), y_scale=float(y_scale), const_features=np.zeros(0),
                x_scaler="custom")


def affine_net(value_lists, hidden, seed: int, y_mean=1.4, y_scale=0.3):
    """Weights for which every hidden pre-activation is positive on the whole space
    (|z| <= 1, b_1 > sum_j |W_1[j,:]|, W_l >= 0 and b_l > 0 for l >= 2), so the net
    is exactly affine in z (SURVEY §4 derived pin 3)."""
    rng = np.random.default_rng([seed, 0xAFF1])
    widths = [len(value_lists)] + list(hidden) + [1]
    W, b = [], []
    for l, (fi, fo) in enumerate(zip(widths[:-1], widths[1:])):
        bound = np.sqrt(6.0 / (fi + fo))
        if l == 0:
            w = rng.uniform(-bound, bound, (fi, fo))
            bb = np.abs(w).sum(axis=0) + rng.uniform(0.05, 0.5, fo)
        elif l < len(widths) - 2:
            w = rng.uniform(0.0, bound, (fi, fo)) / 2.0
            bb = rng.uniform(0.05, 0.5, fo)
        else:
            w = rng.uniform(-bound, bound, (fi, fo))
            bb = rng.uniform(-0.5, 0.5, fo)
        W.append(w)
        b.append(bb)
    shift, scale = _unit_scaler(value_lists)
    return dict(widths=widths, members=[dict(W=W, b=b)], x_shift=shift, x_scale=scale,
                y_mean=float(y_mean), y_scale=float(y_scale), const_features=np.zeros(0),
                x_scaler="custom")


def predict_rows(value_lists, n: int, seed: int) -> np.ndarray:
    """n random raw configs (float64 values from the lists) for surrogate_predict."""
    rng = np.random.default_rng([seed, 0xF00D])
    cols = [np.asarray(v, np.float64)[rng.integers(0, len(v), n)] for v in value_lists]
    return np.stack(cols, axis=1)


# ---------------------------------------------------------------- training inputs
# Seeded inputs of the GPU-training parity tests: both the
# oracle and the CUDA trainer receive the same initial weights (glorot_init),
# the same standardised data (training_rows) and the same epoch orders
# (epoch_permutations); nothing here is the method's arithmetic.

def glorot_init(widths, seed: int):
    """Glorot-uniform U(+-sqrt(6/(fan_in+fan_out))) weights and biases (the
    scikit-learn initialisation the paper's MLPRegressor uses)."""
    rng = np.random.default_rng([seed, 0x61])
    W, b = [], []
    for fi, fo in zip(widths[:-1], widths[1:]):
        bound = np.sqrt(6.0 / (fi + fo))
        W.append(rng.uniform(-bound, bound, (fi, fo)))
        b.append(rng.uniform(-bound, bound, fo))
    return W, b


def training_rows(value_lists, n: int, seed: int, noise: float = 0.02):
    """n random configs and a smooth synthetic runtime (a sum of log2-quadratic
    bowls plus Gaussian noise), both standardised column-wise: (Xs [n, P], ys [n])."""
    X = predict_rows(value_lists, n, seed)
    rng = np.random.default_rng([seed, 0x7A])
    L = np.log2(X)
    opt = np.array([rng.uniform(np.log2(min(v)), np.log2(max(v))) for v in value_lists])
    a = rng.uniform(0.02, 0.1, len(value_lists))
    y = 1.0 + ((L - opt) ** 2 * a).sum(axis=1) + noise * rng.standard_normal(n)
    Xs = (X - X.mean(axis=0)) / np.where(X.std(axis=0) > 0, X.std(axis=0), 1.0)
    ys = (y - y.mean()) / y.std()
    return Xs, ys


def epoch_permutations(n: int, epochs: int, seed: int) -> np.ndarray:
    """[epochs, n] uint32: one seeded permutation of 0..n-1 per epoch."""
    rng = np.random.default_rng([seed, 0x5EF])
    return np.stack([rng.permutation(n) for _ in range(epochs)]).astype(np.uint32)
