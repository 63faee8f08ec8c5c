#!/usr/bin/env python3
"""Full-enumeration oracle top-k of a trained net over a whole space, stored as a
golden file for the GPU parity tests ("cfg 2: full enumeration,
top-16 per G17").  Calls only oracle/ (float64 numpy); the space is split into
contiguous ranges evaluated by worker processes and merged under the same
(t, I) order (oracle.sweep.merge_topk).

    python scripts/make_golden_topk.py cfg2 64      # -> tests/golden/cfg2_full_top64_oracle.json
"""

import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402
from oracle import space as ospace  # noqa: E402
from oracle import sweep as osweep  # noqa: E402


def _work(args):
    name, lo, hi, k = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    wl = workloads.WORKLOADS[name]
    vl = workloads.space(wl.space)
    model = workloads.load_model(wl.weights)
    if wl.device_encoding:  # combined-GPU model: sweep for the bench's target device (G3)
        model = workloads.with_device(model, workloads.device_features(wl.device_encoding, wl.devices[-1]))
    i, t = osweep.topk(model, vl, k, lo, hi)
    return i, t


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    wl = workloads.WORKLOADS[name]
    vl = workloads.space(wl.space)
    N = ospace.cardinality([len(v) for v in vl])
    nproc = os.cpu_count() or 1
    parts = 4 * nproc
    bounds = [(N * p) // parts for p in range(parts + 1)]
    t0 = time.time()
    with mp.Pool(nproc) as pool:
        res = pool.map(_work, [(name, bounds[p], bounds[p + 1], k) for p in range(parts)])
    idx, t = osweep.merge_topk(res, k)
    wpath = os.path.join(ROOT, "weights", wl.weights + ".npz")
    out = {"workload": name, "space": wl.space, "configs": int(N), "k": k, "weights": wl.weights,
           "device": (wl.device_encoding, wl.devices[-1]) if wl.device_encoding else None,
           "weights_sha256": hashlib.sha256(open(wpath, "rb").read()).hexdigest(),
           "made_by": "scripts/make_golden_topk.py (oracle/ only, float64 numpy, full enumeration)",
           "seconds": round(time.time() - t0, 1),
           "idx": [int(i) for i in idx], "t": [float(repr_t) for repr_t in t]}
    path = os.path.join(ROOT, "tests", "golden", f"{name}_full_top{k}_oracle.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path, out["seconds"], "s", out["idx"][:4], out["t"][:4])


if __name__ == "__main__":
    main()
