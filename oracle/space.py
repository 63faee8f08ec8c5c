"""Search-space arithmetic (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

The paper tunes 7 OpenACC kernels x {gang, vector} = 14 parameters,
each with an explicit value list (Table "Tuning Parameters"); the
space is their Cartesian product, |S| = prod_j r_j (10^7 * 12^7).

Index convention ("lexicographic order of value
indices"): parameter 0 is the most significant digit, parameter P-1 the least;

    I = sum_j d_j * prod_{l>j} r_l ,   0 <= d_j < r_j .
"""

from __future__ import annotations

import itertools

import numpy as np


def cardinality(radices) -> int:
    """|S| = product of the value-list lengths, as an exact Python int."""
    n = 1
    for r in radices:
        r = int(r)
        if r < 1:
            raise ValueError("every radix must be >= 1")
        n *= r
    return n


def strides(radices) -> list[int]:
    """stride_j = prod_{l>j} r_l (exact ints); I = sum_j d_j * stride_j."""
    s = [1] * len(radices)
    acc = 1
    for j in range(len(radices) - 1, -1, -1):
        s[j] = acc
        acc *= int(radices[j])
    return s


def decode(idx, radices) -> np.ndarray:
    """Flat index -> digit tuple, least significant parameter last (G10).

    Follows the definition step by step: for j = P-1 ... 0, d_j = I mod r_j,
    I = I div r_j.  ``idx`` is an int or an array of non-negative ints < |S|;
    returns int64 array of shape (..., P).
    """
    idx = np.asarray(idx, dtype=np.uint64)
    n = cardinality(radices)
    if idx.size and int(idx.max()) >= n:
        raise ValueError("index out of range")
    rem = idx.copy()
    out = np.empty(idx.shape + (len(radices),), dtype=np.int64)
    for j in range(len(radices) - 1, -1, -1):
        r = np.uint64(int(radices[j]))
        out[..., j] = (rem % r).astype(np.int64)
        rem = rem // r
    return out


def encode(digits, radices) -> np.ndarray:
    """Digit tuples -> flat index (inverse of decode); Horner form."""
    digits = np.asarray(digits, dtype=np.int64)
    if digits.shape[-1] != len(radices):
        raise ValueError("digit tuple length must equal the number of parameters")
    acc = np.zeros(digits.shape[:-1], dtype=np.uint64)
    for j, r in enumerate(radices):
        d = digits[..., j]
        if np.any(d < 0) or np.any(d >= int(r)):
            raise ValueError("digit out of range")
        acc = acc * np.uint64(int(r)) + d.astype(np.uint64)
    return acc


def values_of(digits, value_lists) -> np.ndarray:
    """x_j = v_j[d_j] (Table "Tuning Parameters"), as float64 of shape (..., P)."""
    digits = np.asarray(digits, dtype=np.int64)
    out = np.empty(digits.shape, dtype=np.float64)
    for j, vals in enumerate(value_lists):
        out[..., j] = np.asarray(vals, dtype=np.float64)[digits[..., j]]
    return out


def enumerate_all(value_lists, cap: int = 10**6):
    """Every config once, lexicographic in value indices; size <= cap."""
    n = cardinality([len(v) for v in value_lists])
    if n > cap:
        raise ValueError(f"space of {n} configs exceeds enumeration cap {cap}")
    return [tuple(c) for c in itertools.product(*[list(v) for v in value_lists])]


def check_value_lists(value_lists) -> None:
    """Each list non-empty, strictly increasing, all > 0."""
    if len(value_lists) == 0:
        raise ValueError("at least one parameter")
    for vals in value_lists:
        v = list(vals)
        if len(v) == 0 or any(x <= 0 for x in v) or any(b <= a for a, b in zip(v, v[1:])):
            raise ValueError("value lists must be non-empty, strictly increasing, > 0")


def sample_indices(radices, n: int, rng: np.random.Generator) -> np.ndarray:
    """n distinct configs, each digit drawn i.i.d. uniform ("systematic random
    sampling"); exact duplicates are discarded and redrawn, at most 100*n
    draws.  Returns the flat indices in draw order (uint64)."""
    size = cardinality(radices)
    if n > size:
        raise ValueError("space has fewer than n distinct configs")
    seen: set[int] = set()
    order: list[int] = []
    draws = 0
    st = strides(radices)
    while len(order) < n:
        if draws >= 100 * max(n, 1):
            raise RuntimeError("sampling exhausted 100*n draws")
        m = n - len(order)
        digits = np.stack([rng.integers(0, int(r), size=m) for r in radices], axis=1)
        draws += m
        for row in digits:
            i = sum(int(d) * s for d, s in zip(row, st))
            if i not in seen:
                seen.add(i)
                order.append(i)
                if len(order) == n:
                    break
    return np.array(order, dtype=np.uint64)


def split(n_rows: int, train_fraction: float, rng: np.random.Generator):
    """Seeded shuffle then split, train size = round(fraction * N) (
    P:307 "10,000 samples, with 7,500 allocated for training")."""
    if not (0.0 < train_fraction < 1.0):
        raise ValueError("0 < train_fraction < 1")
    if n_rows < 2:
        raise ValueError("need at least 2 rows")
    perm = rng.permutation(n_rows)
    n_train = int(round(train_fraction * n_rows))
    return perm[:n_train], perm[n_train:]


def shard(n: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous shard [lo, hi) of [0, n) for rank r of W:
    q = n // W, rem = n % W, lo = r*q + min(r, rem)."""
    q, rem = divmod(int(n), int(world))
    lo = rank * q + min(rank, rem)
    hi = lo + q + (1 if rank < rem else 0)
    return lo, hi
