"""Feature centring and scaling (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

P:271-273: "we employ the StandardScaler" (mean removal and variance scaling).
scikit-learn's StandardScaler uses the population standard deviation (ddof=0)
and maps a (near-)zero scale to 1 (``_handle_zeros_in_scale``), so a constant
column transforms to 0.  Reading G1: the north star's
"min-max" is served by the same affine form with shift = min, scale = max - min.
"""

from __future__ import annotations

import numpy as np


def _handle_zeros(scale: np.ndarray) -> np.ndarray:
    eps = 10.0 * np.finfo(np.float64).eps
    scale = np.array(scale, dtype=np.float64, copy=True)
    scale[scale < eps] = 1.0
    return scale


def fit_standard(X) -> tuple[np.ndarray, np.ndarray]:
    """(mean, scale) per column: mean, population std with zero -> 1."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[0] == 0:
        raise ValueError("X must be a non-empty 2-D array")
    mean = X.mean(axis=0)
    std = np.sqrt(((X - mean) ** 2).mean(axis=0))
    return mean, _handle_zeros(std)


def fit_minmax(X) -> tuple[np.ndarray, np.ndarray]:
    """(shift, scale) = (min, max - min) per column, zero range -> 1 (G1)."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[0] == 0:
        raise ValueError("X must be a non-empty 2-D array")
    lo = X.min(axis=0)
    return lo, _handle_zeros(X.max(axis=0) - lo)


def transform(X, shift, scale) -> np.ndarray:
    """z = (x - shift) / scale, column-wise."""
    X = np.asarray(X, dtype=np.float64)
    if X.shape[-1] != len(shift):
        raise ValueError("column count does not match the scaler")
    return (X - shift) / scale


def inverse(Z, shift, scale) -> np.ndarray:
    """x = z * scale + shift."""
    return np.asarray(Z, dtype=np.float64) * scale + shift
