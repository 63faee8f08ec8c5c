#!/usr/bin/env python3
"""Explicit-batch throughput of surrogate_predict (SPEC-style
sampled search feeds rows from HBM, 56 B per row in).  Prints one JSON line in
bench.py's format (metric: predicted rows/s).

    python scripts/bench_predict.py [--workload cfg2] [--rows 16777216] [--steps 10] [--warmup 3]
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
from bench import PEAK_RATIO, algorithmic_flops, load_peaks  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--rows", type=int, default=1 << 24)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--precision", default=None)
a = ap.parse_args()
wl = workloads.WORKLOADS[a.workload]
vl = workloads.space(wl.space)
model = workloads.load_model(wl.weights)
if wl.device_encoding:
    model = workloads.with_device(model, workloads.device_features(wl.device_encoding, wl.devices[-1]))
prec = a.precision or wl.precision
h = pk.Surrogate(0).load(model, prec)
# random configs of the space (raw values), generated on the host once: the rows a sampler would produce
rng = np.random.default_rng(7)
N = int(np.prod([len(v) for v in vl]))
idx = rng.integers(0, N, a.rows, dtype=np.uint64)
d = []
rem = idx.copy()
for r in reversed([len(v) for v in vl]):
    d.append(rem % np.uint64(r))
    rem //= np.uint64(r)
digits = np.stack(d[::-1], 1)
X = np.stack([np.asarray(vl[j], np.float32)[digits[:, j].astype(np.int64)] for j in range(len(vl))], 1)
x = torch.from_numpy(X).cuda()
xh = torch.from_numpy(X).pin_memory()
t = torch.empty(a.rows, dtype=torch.float32, device="cuda")
for _ in range(a.warmup):
    t = h.predict(x)
torch.cuda.synchronize()
h.kernel_timing(True)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
for s in range(a.steps):
    ev[s][0].record()
    t = h.predict(x)
    ev[s][1].record()
torch.cuda.synchronize()
ms = sum(e0.elapsed_time(e1) for e0, e1 in ev) / a.steps
k1_ms, k1_n = h.kernel_timing_get()
h.kernel_timing(False)
# end to end: rows H2D from pinned memory, predict, times D2H
th = torch.empty(a.rows, dtype=torch.float32).pin_memory()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    x.copy_(xh, non_blocking=True)
    tt = h.predict(x)
    th.copy_(tt, non_blocking=True)
e1.record()
torch.cuda.synchronize()
e2e_ms = e0.elapsed_time(e1) / a.steps
burst, sustained, src = load_peaks()
flops = algorithmic_flops(model["widths"]) * len(model["members"]) * a.rows
k1_step = k1_ms / a.steps
print(json.dumps({
    "metric": "surrogate_predict rows/s (explicit batch from HBM)", "value": a.rows / (ms / 1e3), "unit": "rows/s",
    "n_gpus": 1, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
    "dtype": prec, "data": "synthetic",
    "config": {"workload": wl.name, "rows": a.rows, "row_bytes_in": 4 * X.shape[1], "row_bytes_out": 4},
    "roofline": {"bound": "tensor", "achieved": flops / (k1_step / 1e3) / 1e12,
                 "peak": burst * PEAK_RATIO[h.arith()[0]], "unit": "TFLOP/s",
                 "frac": flops / (k1_step / 1e3) / 1e12 / (burst * PEAK_RATIO[h.arith()[0]]),
                 "hbm_GBps": a.rows * (4 * X.shape[1] + 4) / (k1_step / 1e3) / 1e9},
    "e2e": {"value": a.rows / (e2e_ms / 1e3), "unit": "rows/s", "h2d_bytes_per_step": int(X.nbytes),
            "d2h_bytes_per_step": int(4 * a.rows)}}))
