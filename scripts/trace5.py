import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_14011_b200 as pk
import workloads
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
wl = workloads.WORKLOADS["cfg2"]
vl = workloads.space(wl.space)
h = pk.Surrogate(0).load(workloads.load_model(wl.weights), prec)
h.sweep(vl, 16)
buf = torch.zeros(64 * 4 * 16, dtype=torch.int64, device="cuda")
h.debug_trace(buf)
h.sweep(vl, 16)
torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(64, 4, 16).astype(np.float64)
for s in range(2):  # slot (trace rows of sub 0)
    d = t[10:40, s]
    if d[:, 0].min() <= 0: continue
    print("slot", s, "cycles per tile", np.median(np.diff(d[:, 0])))
    for a, b, lab in [(0, 1, "wait L1"), (1, 2, "epi1"), (2, 3, "L2 (issue..done)"), (3, 5, "final"), (5, 6, "A0+issue L1 / bar")]:
        print(f"   {lab:20s} {np.median(d[:, b] - d[:, a]):8.0f}")
d = t[10:40, 0]
print("raw events (cycles after loop top) for 3 tiles:")
for j in range(3):
    print([int(x - d[j, 0]) for x in d[j, :7]])
