"""Independent expected results used as pins (not the oracle, not the CUDA path).

* ``brute_times``  — pure-Python loops over configs for tiny spaces (brute force);
* ``affine_kbest`` — exact k-best of an affine net by best-first enumeration of
  a separable sum (SURVEY §4 derived pin 3): no sweep at all, so it pins the
  sweep's top-k at any size, including 1.35e10 configs.
"""

from __future__ import annotations

import heapq
import itertools

import numpy as np


def brute_times(model, value_lists):
    """t(I) for every config, plain Python floats, lexicographic order."""
    Ws = [[[float(x) for x in row] for row in w] for w in model["members"][0]["W"]]
    bs = [[float(x) for x in v] for v in model["members"][0]["b"]]
    sh = [float(x) for x in model["x_shift"]]
    sc = [float(x) for x in model["x_scale"]]
    out = []
    for cfg in itertools.product(*value_lists):
        h = [(float(x) - sh[j]) / sc[j] for j, x in enumerate(cfg)]
        for l, (W, b) in enumerate(zip(Ws, bs)):
            nxt = []
            for o in range(len(b)):
                s = b[o]
                for i in range(len(h)):
                    s += h[i] * W[i][o]
                nxt.append(s if l == len(Ws) - 1 or s > 0.0 else 0.0)
            h = nxt
        out.append(model["y_mean"] + model["y_scale"] * h[0])
    return out


def affine_tables(model, value_lists):
    """For a net whose hidden units never switch off: t = C + sum_j T_j[d_j]."""
    m = model["members"][0]
    c = np.eye(len(value_lists))
    c0 = np.zeros(1)
    prod = None
    for W, b in zip(m["W"], m["b"]):
        prod = W if prod is None else prod @ W
    # constant term: b_1 W_2..W_L + b_2 W_3..W_L + ... + b_L
    c0 = np.zeros(m["b"][-1].shape)
    for l, b in enumerate(m["b"]):
        term = b
        for W in m["W"][l + 1:]:
            term = term @ W
        c0 = c0 + term
    coef = (c @ prod)[:, 0]
    C = model["y_mean"] + model["y_scale"] * float(c0[0])
    tables = []
    for j, vals in enumerate(value_lists):
        z = (np.asarray(vals, np.float64) - model["x_shift"][j]) / model["x_scale"][j]
        tables.append(model["y_scale"] * coef[j] * z)
    return C, tables


def affine_kbest(model, value_lists, k: int, extra: int = 64):
    """(idx list, t list) of the k best configs, ordered by (t, idx), via best-first
    search over rank vectors (each state from its unique parent: successors
    increment coordinates j >= the last non-zero coordinate)."""
    C, tables = affine_tables(model, value_lists)
    P = len(tables)
    order = [np.argsort(t, kind="stable") for t in tables]
    srt = [t[o] for t, o in zip(tables, order)]
    radices = [len(v) for v in value_lists]
    strides = [1] * P
    for j in range(P - 2, -1, -1):
        strides[j] = strides[j + 1] * radices[j + 1]
    start = (0,) * P
    heap = [(sum(float(s[0]) for s in srt), start, 0)]
    got = []
    while heap and len(got) < k + extra:
        val, st, p = heapq.heappop(heap)
        digits = [int(order[j][st[j]]) for j in range(P)]
        idx = sum(d * s for d, s in zip(digits, strides))
        got.append((C + val, idx))
        for j in range(p, P):
            if st[j] + 1 < radices[j]:
                ns = list(st)
                ns[j] += 1
                nv = val - float(srt[j][st[j]]) + float(srt[j][st[j] + 1])
                heapq.heappush(heap, (nv, tuple(ns), j))
    got.sort()
    got = got[:k]
    return [i for _, i in got], [t for t, _ in got]
