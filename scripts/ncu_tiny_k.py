#!/usr/bin/env python3
"""ncu target: a shard of one tile per CTA slot (148 x 4 x 128 configs) of cfg5
at k = 1024: the sweep's fixed cost (list fill, per-CTA lists, merge tree)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_14011_b200 as pk  # noqa: E402
import workloads  # noqa: E402
k = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
wl = workloads.WORKLOADS["cfg5"]
vl = workloads.space(wl.space)
h = pk.Surrogate(0).load(workloads.load_model(wl.weights), "fp16")
for _ in range(2):
    idx, t, _ = h.sweep(vl, k, 5_000_000_000, 5_000_000_000 + 148 * 4 * 128)
torch.cuda.synchronize()
print(int(idx[0]), float(t[0]))
