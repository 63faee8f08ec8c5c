"""Exhaustive surrogate sweep and top-k (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

The plain definition the GPU path must reproduce:

    d_j(I) mixed-radix digits (space.decode), x_j(I) = v_j[d_j(I)]
    z = (x - shift) / scale                       (StandardScaler)
    t(I) = (1/E) sum_e (mu_y + sigma_y * yhat_e(z))
    TopK(R) = the k smallest (t(I), I) over I in R under lexicographic order on
              (t, I), NaN ranked after +inf, sorted ascending (G10, G13).

The paper never says how the trained model is searched ("the model
consistently identifies configurations with the lowest runtime"); reading G13
takes the exhaustive sweep.  Chunking over I only bounds memory: every row is
computed independently in float64 exactly as mlp.predict does.
"""

from __future__ import annotations

import numpy as np

from . import mlp as _mlp
from . import space as _space


def times(model, value_lists, begin: int, end: int) -> np.ndarray:
    """t(I) for I in [begin, end), float64."""
    radices = [len(v) for v in value_lists]
    idx = np.arange(begin, end, dtype=np.uint64)
    return _mlp.predict(model, _space.values_of(_space.decode(idx, radices), value_lists))


def times_at(model, value_lists, idx) -> np.ndarray:
    """t(I) at explicit indices (sampled parity checks)."""
    radices = [len(v) for v in value_lists]
    idx = np.asarray(idx, dtype=np.uint64)
    return _mlp.predict(model, _space.values_of(_space.decode(idx, radices), value_lists))


def _order(t: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """Permutation sorting by (t, I); numpy sorts NaN after +inf."""
    return np.lexsort((idx, t))


def topk(model, value_lists, k: int, begin: int = 0, end: int | None = None,
         chunk: int = 1 << 20):
    """(idx uint64[count], t float64[count]) of the k best in [begin, end),
    count = min(k, end - begin) (G18)."""
    if k < 1:
        raise ValueError("k >= 1")
    radices = [len(v) for v in value_lists]
    if end is None:
        end = _space.cardinality(radices)
    best_i = np.zeros(0, dtype=np.uint64)
    best_t = np.zeros(0, dtype=np.float64)
    for lo in range(begin, end, chunk):
        hi = min(end, lo + chunk)
        t = times(model, value_lists, lo, hi)
        i = np.arange(lo, hi, dtype=np.uint64)
        ci = np.concatenate([best_i, i])
        ct = np.concatenate([best_t, t])
        o = _order(ct, ci)[:k]
        best_i, best_t = ci[o], ct[o]
    return best_i, best_t


def merge_topk(lists, k: int):
    """Top-k of the union of several (idx, t) lists under the same order (G17 merge)."""
    ci = np.concatenate([np.asarray(i, np.uint64) for i, _ in lists])
    ct = np.concatenate([np.asarray(t, np.float64) for _, t in lists])
    o = _order(ct, ci)[:k]
    return ci[o], ct[o]
