#!/usr/bin/env python3
"""Dump CTA 0's pipeline timeline of one sweep (development aid)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_14011_b200 as pk
import workloads
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
wl = workloads.WORKLOADS[name]
vl = workloads.space(wl.space)
prec = sys.argv[2] if len(sys.argv) > 2 else "fp16"
h = pk.Surrogate(0).load(workloads.load_model(wl.weights), prec)
h.sweep(vl, wl.k)
buf = torch.zeros(64 * 4 * 16, dtype=torch.int64, device="cuda")
h.debug_trace(buf)
h.sweep(vl, wl.k)
torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(64, 4, 16)
t0 = t[t > 0].min()
names = ["L1", "wD1", "epi1", "wD2a", "finA", "wD2b", "finB", "topk", "", "", "", "", "", "", "", ""]
for j in range(20, 24):
    for s in range(4):
        row = t[j, s]
        print(f"round {j} slot {s}: " + " ".join(f"{names[e]}={row[e]-t0}" for e in range(16) if row[e] > 0))
# steady-state per-tile stats
d = t[10:50, :4].astype(np.float64)
per_round = np.diff(d[:, 0, 0])
print("cycles per round (4 tiles):", np.median(per_round), "-> per tile", np.median(per_round) / 4)
for a, b, lab in [(0, 1, "issueL1->wD1"), (1, 2, "epi1"), (2, 3, "issueL2a->wD2a"), (3, 4, "finA"),
                  (4, 5, "issueL2b->wD2b"), (5, 6, "finB"), (6, 7, "topk"), (7, 0, "topk->next arrA0")]:
    x = d[:, :, b] - d[:, :, a] if lab != "topk->next arrA0" else d[1:, :, 0] - d[:-1, :, 7]
    print(f"{lab:18s} median {np.median(x):8.0f}")
