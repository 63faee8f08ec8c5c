#!/usr/bin/env python3
"""Minimal launch sequence for an ncu capture: 2 sweeps of one workload/precision
(profile the second K1 launch with `-k regex:sweep_kernel -s 1 -c 1`)."""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_14011_b200 as pk  # noqa: E402
import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
wl = workloads.WORKLOADS[name]
vl = workloads.space(wl.space)
model = workloads.load_model(wl.weights)
if wl.device_encoding:  # combined-training model: one target device (G3)
    model = workloads.with_device(model, workloads.device_features(wl.device_encoding, wl.devices[-1]))
h = pk.Surrogate(0).load(model, prec)
for _ in range(2):
    idx, t, _ = h.sweep(vl, wl.k)
torch.cuda.synchronize()
print(name, prec, int(idx[0]), float(t[0]))
