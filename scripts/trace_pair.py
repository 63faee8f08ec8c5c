#!/usr/bin/env python3
"""Pipeline timeline of CTA 0 in the CTA-pair kernel (development aid; needs
a SURR_EXTRA_FLAGS=-DSURR_TRACE build)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_14011_b200 as pk
import workloads
wl = workloads.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
vl = workloads.space(wl.space)
h = pk.Surrogate(0).load(workloads.load_model(wl.weights), "bf16")
h.sweep(vl, wl.k)
buf = torch.zeros(200 * 4 * 16, dtype=torch.int64, device="cuda")
h.debug_trace(buf)
h.sweep(vl, wl.k)
torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(200, 4, 16).astype(np.float64)
names = {0: ["A0F", "RF", "aq0", "aq1", "aq2", "aq3", "bq0", "bq1", "bq2", "bq3", "DBw", "L1iss"],
         1: ["wD1", "Q0", "Q1", "wD2", "Q0", "Q1", "wD3", "", "", "fin", "bar1", "bar2", "w1start"],
         2: ["wD1", "Q2", "Q3", "wD2", "Q2", "Q3", "wD3", "", "", "fin", "bar1", "bar2", "w1start"],
         3: ["A0E", "A0F"]}
base = t[100, 0, 0]
for j in range(100, 103):
    for s in range(4):
        print(f"tile {j} {['issuer', 'sub0', 'sub1', 'prod'][s]:6s}: " +
              " ".join(f"{n}={t[j, s, e] - base:.0f}" for e, n in enumerate(names[s]) if n and t[j, s, e] > 0))
per = np.diff(t[20:180, 0, 0])
print("cycles per tile (median):", np.median(per))
ev = [(0, 0, "A0F(L1 issue)"), (1, 0, "sub0 wD1"), (0, 2, "aq0 (L2 Q0 issue)"), (0, 5, "aq3"),
      (1, 3, "sub0 wD2"), (2, 3, "sub1 wD2"), (0, 6, "bq0 (L3 Q0 issue)"), (0, 9, "bq3"), (1, 6, "sub0 wD3"),
      (2, 6, "sub1 wD3"), (0, 10, "DB wait done"), (1, 9, "sub0 fin"), (2, 9, "sub1 fin"), (1, 10, "bar1"),
      (1, 11, "bar2")]
d = t[20:180]
for s, e, lab in ev:
    print(f"{lab:20s} {np.median(d[:, s, e] - d[:, 0, 0]):8.0f}")
