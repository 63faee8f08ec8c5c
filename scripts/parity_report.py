#!/usr/bin/env python3
"""Measured parity of the CUDA path against the float64 oracle, per workload
and precision (development evidence beside the -m gpu tests, which assert the
bounds): max / 99.9th-percentile relative error of t over seeded
random slices of the space in the bench's launch configuration (dense mode of
the same kernel), the north star's bound, and for cfg2 the whole-space top-64
against the oracle's full float64 enumeration (tests/golden, written by
scripts/make_golden_topk.py from oracle/ only).  Prints one JSON line per row.

    python scripts/parity_report.py [--slices 8] [--slice 65536]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_14011_b200 as pk  # noqa: E402
import workloads  # noqa: E402
from oracle import sweep as osweep  # noqa: E402
from tests.helpers import TOL, rel_err  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--slices", type=int, default=8)
ap.add_argument("--slice", type=int, default=1 << 16)
a = ap.parse_args()

rows = []
for wl_name in ("cfg2", "cfg5", "cfg3"):
    wl = workloads.WORKLOADS[wl_name]
    vl = workloads.space(wl.space)
    model = workloads.load_model(wl.weights)
    N = int(np.prod([len(v) for v in vl], dtype=object))
    rng = np.random.default_rng(0x2306014011 + len(wl_name))
    starts = sorted(int(x) for x in rng.integers(0, N - a.slice, a.slices))
    ref = {s0: osweep.times(model, vl, s0, s0 + a.slice) for s0 in starts}
    for prec in (("fp16", "bf16", "fp32") if wl_name != "cfg3" else ("fp16", "bf16")):
        h = pk.Surrogate(0).load(model, prec)
        errs = []
        for s0 in starts:
            d = h.eval_range(vl, s0, s0 + a.slice)
            torch.cuda.synchronize()
            errs.append(rel_err(d.cpu().numpy(), ref[s0], model["y_scale"]))
        e = np.concatenate(errs)
        rows.append({"workload": wl_name, "net": "-".join(map(str, model["widths"])), "precision": prec,
                     "configs": int(e.size), "max_rel": float(e.max()),
                     "p999_rel": float(np.quantile(e, 0.999)), "bound": TOL[prec],
                     "within": bool(e.max() <= TOL[prec])})
        h.close()
        print(json.dumps(rows[-1]), flush=True)

# cfg2 whole space: top-64 vs the oracle's float64 enumeration
gold = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "tests", "golden", "cfg2_full_top64_oracle.json")))
wl = workloads.WORKLOADS["cfg2"]
vl = workloads.space(wl.space)
model = workloads.load_model(wl.weights)
g_idx = [int(x) for x in gold["idx"]]
for prec in ("fp16", "bf16", "fp32"):
    h = pk.Surrogate(0).load(model, prec)
    idx, t, _ = h.sweep(vl, 64)
    torch.cuda.synchronize()
    gi = [int(x) for x in idx.cpu().numpy()]
    rows.append({"workload": "cfg2 whole space", "precision": prec, "k": 64,
                 "same_set_as_oracle": set(gi) == set(g_idx), "same_order": gi == g_idx,
                 "common": len(set(gi) & set(g_idx)), "top1_equal": gi[0] == g_idx[0]})
    h.close()
    print(json.dumps(rows[-1]), flush=True)
