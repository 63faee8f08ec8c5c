#!/usr/bin/env python3
"""CTA 0 timeline of the 3xFP16 FP32-path kernel (development aid; needs a
-DSURR_TRACE build: SURR_EXTRA_FLAGS=-DSURR_TRACE).  Rows: slot s, sub q."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_14011_b200 as pk
import workloads
wl = workloads.WORKLOADS["cfg2"]
vl = workloads.space(wl.space)
h = pk.Surrogate(0).load(workloads.load_model(wl.weights), "fp32")
h.sweep(vl, 16)
buf = torch.zeros(64 * 4 * 16, dtype=torch.int64, device="cuda")
h.debug_trace(buf)
h.sweep(vl, 16)
torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(64, 4, 16).astype(np.float64)
names = ["top", "L1done", "epi1", "L2a_iss", "L2a_done", "partA", "L2b_done", "partB", "redbar", "emit"]
t0 = t[t > 0].min()
for j in range(20, 24):
    for sq in range(4):
        row = t[j, sq]
        print(f"tile {j} s{sq % 2} q{sq // 2}: " + " ".join(f"{names[e]}={int(row[e] - t0)}" for e in range(10) if row[e] > 0))
for sq in range(4):
    d = t[10:50, sq]
    print(f"s{sq % 2} q{sq // 2} cycles/tile {np.median(np.diff(d[:, 0])):.0f}: " +
          " ".join(f"{names[e - 1]}->{names[e]} {np.median(d[:, e] - d[:, e - 1]):.0f}" for e in range(1, 10) if d[:, e].min() > 0))
