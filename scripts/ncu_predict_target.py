#!/usr/bin/env python3
"""Minimal launch sequence for an ncu capture of the explicit-batch predict kernel (K3)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_14011_b200 as pk  # noqa: E402
import workloads  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp16"
vl = workloads.space("cfg2")
h = pk.Surrogate(0).load(workloads.load_model("cfg2_14-128-128-1"), prec)
X = torch.tensor(workloads.predict_rows(vl, 1 << 22, seed=1), dtype=torch.float32, device="cuda:0")
for _ in range(2):
    t = h.predict(X)
torch.cuda.synchronize()
print(float(t[:8].sum()))
