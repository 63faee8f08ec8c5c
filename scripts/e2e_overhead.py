#!/usr/bin/env python3
"""Per-call host overhead of surrogate_sweep_host (the e2e call) vs the device
time of the same sweep: small and full ranges (development aid; SURR_LIB selects
the library)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_14011_b200 as pk
import workloads
vl = workloads.space("cfg2")
h = pk.Surrogate(0).load(workloads.load_model("cfg2_14-128-128-1"), "fp16")
for n in (1 << 16, 1 << 22, 170859375):
    d = pk.SpaceDesc(vl, 0, n)
    out = (np.empty(16, np.uint64), np.empty(16, np.float32))
    for _ in range(3):
        h.sweep_host(vl, 16, desc=d, out=out)
    t0 = time.perf_counter()
    for _ in range(20):
        h.sweep_host(vl, 16, desc=d, out=out)
    host = (time.perf_counter() - t0) / 20
    idx = torch.empty(16, dtype=torch.int64, device="cuda"); tt = torch.empty(16, dtype=torch.float32, device="cuda")
    for _ in range(3):
        h.sweep_into(d, 16, idx, tt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        h.sweep_into(d, 16, idx, tt)
    e1.record(); torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) / 20 / 1e3
    print(f"{os.environ.get('SURR_LIB', 'current')} n={n}: sweep_host {host*1e6:9.1f} us  device {dev*1e6:9.1f} us  overhead {(host-dev)*1e6:8.1f} us")
