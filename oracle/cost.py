"""Synthetic solver-time surface (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

The paper's labels are measured SENSEI solver times on real GPUs, normalised
into [0.8 s, 2.0 s] by choosing the iteration count per GPU; those
measurements are out of scope.  This module is the seeded
stand-in SPEC.md's ``synthetic_cost`` describes:

    t = base + sum_k [A_k log2^2(g_k/g*_k) + B_k log2^2(v_k/v*_k)]
             + c_int * sum_k log2(g_k/g*_k) log2(v_k/v*_k) + noise

with kernel k's gang at parameter 2k and vector at 2k+1 (Table order).
Reading G19: every device's surface is calibrated independently so
that the noiseless values span exactly [0.8, 2.0] s over the space:
t = 0.8 + 1.2 (Q - Q_min) / (Q_max - Q_min) + noise, Q the bracketed sum.
Noise is Gaussian, sigma = 0.02 s by default, a pure function of
(index, device, seed) via a SplitMix64 hash and Box-Muller.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import space as _space

# Table "GPU specification": double-precision GFLOPS.
DEVICE_GFLOPS = {"C2075": 513.0, "P100": 4700.0, "V100": 7500.0}
T_LO, T_HI = 0.8, 2.0  # P:298 "[0.8 s, 2.0 s]"

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser over a uint64 array (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def _u01(bits: np.ndarray) -> np.ndarray:
    """uniform double in (0, 1]: ((x >> 11) + 1) * 2^-53."""
    return ((bits >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)


@dataclass
class CostModel:
    """One device's calibrated surface over one space."""

    value_lists: list
    g_opt: np.ndarray  # (K,) gang optima (real, inside the value range)
    v_opt: np.ndarray  # (K,) vector optima
    A: np.ndarray      # (K,) curvature amplitudes (raw, before calibration)
    B: np.ndarray
    c_int: float
    q_min: float
    q_max: float
    noise_sigma: float
    seed: int
    device_id: int

    def q(self, values: np.ndarray) -> np.ndarray:
        """The bracketed sum Q for raw values (..., 2K)."""
        g = values[..., 0::2]
        v = values[..., 1::2]
        x = np.log2(g / self.g_opt)
        y = np.log2(v / self.v_opt)
        return (self.A * x * x + self.B * y * y + self.c_int * x * y).sum(axis=-1)

    def noiseless(self, values: np.ndarray) -> np.ndarray:
        q = self.q(values)
        return T_LO + (T_HI - T_LO) * (q - self.q_min) / (self.q_max - self.q_min)

    def noise(self, idx: np.ndarray) -> np.ndarray:
        if self.noise_sigma == 0.0:
            return np.zeros(np.shape(idx))
        key = np.uint64((self.seed * 0x100000001B3 + self.device_id * 0x9E37) & 0xFFFFFFFFFFFFFFFF)
        with np.errstate(over="ignore"):
            h1 = splitmix64(np.asarray(idx, dtype=np.uint64) * np.uint64(2) ^ key)
            h2 = splitmix64(h1 ^ np.uint64(0xD1B54A32D192ED03))
        u1, u2 = _u01(h1), _u01(h2)
        return self.noise_sigma * np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)

    def cost(self, idx: np.ndarray) -> np.ndarray:
        """Solver time in seconds for flat indices (decoded with space.decode)."""
        radices = [len(v) for v in self.value_lists]
        vals = _space.values_of(_space.decode(idx, radices), self.value_lists)
        return self.noiseless(vals) + self.noise(idx)


def _kernel_extrema(vals_g, vals_v, g_opt, v_opt, a, b, c):
    """min and max of A x^2 + B y^2 + c x y over one kernel's 2-D grid (brute force)."""
    x = np.log2(np.asarray(vals_g, dtype=np.float64) / g_opt)[:, None]
    y = np.log2(np.asarray(vals_v, dtype=np.float64) / v_opt)[None, :]
    t = a * x * x + b * y * y + c * x * y
    return float(t.min()), float(t.max())


def make_cost_model(value_lists, seed: int, device: str = "P100", noise_sigma: float = 0.02,
                    c_int_scale: float = 0.5, optima=None) -> CostModel:
    """Draw a surface for one device and calibrate it into [0.8, 2.0] s (G19).

    Optima are log-uniform inside each parameter's [min, max] (or given as a
    (K, 2) array); A_k, B_k ~ U(0.5, 1.5); c_int = u * min_k sqrt(A_k B_k),
    u ~ U(-c_int_scale, c_int_scale), so every kernel's quadratic form stays
    positive definite for c_int_scale < 1 (parity unpinned: the draw itself is
    a modelling choice, only its calibration and optimum are pinned)."""
    if len(value_lists) % 2:
        raise ValueError("parameters come in (gang, vector) pairs")
    K = len(value_lists) // 2
    dev_id = sorted(DEVICE_GFLOPS).index(device) if device in DEVICE_GFLOPS else 99
    rng = np.random.default_rng([seed, dev_id, 0xC057])
    if optima is None:
        lo = np.array([math.log2(v[0]) for v in value_lists])
        hi = np.array([math.log2(v[-1]) for v in value_lists])
        opt = 2.0 ** rng.uniform(lo, hi)
    else:
        opt = np.asarray(optima, dtype=np.float64).reshape(-1)
        _ = rng.uniform(size=len(value_lists))
    g_opt, v_opt = opt[0::2].copy(), opt[1::2].copy()
    A = rng.uniform(0.5, 1.5, size=K)
    B = rng.uniform(0.5, 1.5, size=K)
    c = float(rng.uniform(-c_int_scale, c_int_scale) * np.sqrt(A * B).min())
    q_min = q_max = 0.0
    for k in range(K):
        lo_k, hi_k = _kernel_extrema(value_lists[2 * k], value_lists[2 * k + 1],
                                     g_opt[k], v_opt[k], A[k], B[k], c)
        q_min += lo_k
        q_max += hi_k
    return CostModel(list(value_lists), g_opt, v_opt, A, B, c, q_min, q_max,
                     float(noise_sigma), int(seed), dev_id)
