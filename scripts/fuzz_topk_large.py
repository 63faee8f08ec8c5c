#!/usr/bin/env python3
"""Randomized large-k top-k checks on the B200 (development confidence runs):
random nets / spaces as in tests/test_gpu_fuzz.py, k in 300..1024 and ranges up
to 3e6 configs, GPU top-k vs the oracle's (G17), every precision.

    python scripts/fuzz_topk_large.py [first_seed] [last_seed]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_14011_b200 as pk  # noqa: E402
import workloads  # noqa: E402
from oracle import space as ospace  # noqa: E402
from oracle import sweep as osweep  # noqa: E402
from tests.helpers import TOL, check_topk  # noqa: E402
from tests.test_gpu_fuzz import _case  # noqa: E402

lo = int(sys.argv[1]) if len(sys.argv) > 1 else 0
hi = int(sys.argv[2]) if len(sys.argv) > 2 else 100
bad, ran = [], 0
for seed in range(lo, hi):
    vl, hidden, prec, rng = _case(seed + 10_000)
    model = workloads.random_net(vl, hidden, seed=seed + 200)
    try:
        h = pk.Surrogate(0).load(model, prec)
    except pk.SurrogateError:
        continue
    N = ospace.cardinality([len(v) for v in vl])
    b = int(rng.integers(0, max(1, N // 4)))
    e = int(min(N, b + rng.integers(1, 3_000_000)))
    k = int(min(e - b, rng.integers(300, 1025)))
    try:
        idx, t, cnt = h.sweep(vl, k, b, e)
        ri, rt = osweep.topk(model, vl, k, b, e)
        check_topk(idx.cpu().numpy()[:cnt].astype(np.uint64), t.cpu().numpy()[:cnt], ri, rt,
                   lambda i: osweep.times_at(model, vl, i), TOL[prec], model["y_scale"])
        ran += 1
    except Exception as ex:  # noqa: BLE001
        bad.append((seed, prec, hidden, len(vl), k, b, e, repr(ex)[:200]))
print(f"seeds {lo}..{hi - 1}: {ran} checked, {len(bad)} failures")
for x in bad[:20]:
    print(x)
