#!/usr/bin/env python3
"""CTA 0 timeline of the warp-specialised K1 (sweep_kernel7, -DSURR_TRACE build).
Events per (round, slot): 0 FW loop top (L1 of this tile issued earlier), 1 CW woke
on D1, 2 CW issued L2a, 3 FW woke on D2a, 4 FW done half a + next A0, 5 FW woke
on D2b, 6 FW issued next L1, 7 FW done half b + top-k."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_14011_b200 as pk
import workloads
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
wl = workloads.WORKLOADS[name]
vl = workloads.space(wl.space)
h = pk.Surrogate(0).load(workloads.load_model(wl.weights), sys.argv[2] if len(sys.argv) > 2 else "fp16")
h.sweep(vl, wl.k)
buf = torch.zeros(64 * 4 * 16, dtype=torch.int64, device="cuda")
h.debug_trace(buf)
h.sweep(vl, wl.k)
torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(64, 4, 16).astype(np.float64)
t0 = t[t > 0].min()
for j in range(20, 23):
    for s in range(4):
        print(f"round {j} slot {s}: " + " ".join(f"{e}={int(t[j, s, e] - t0)}" for e in range(8) if t[j, s, e] > 0))
d = t[10:50]
print("cycles per round (4 tiles):", np.median(np.diff(d[:, 0, 0])), "-> per tile", np.median(np.diff(d[:, 0, 0])) / 4)
lab = {(0, 1): "L1 issue->CW woke", (1, 2): "CW epi1+issue L2a", (2, 3): "L2a->FW woke", (3, 4): "FW ldA+L2b+halfA+A0",
       (4, 5): "wait D2b", (5, 6): "ldB+issue L1", (6, 7): "halfB+topk"}
for (a, b), l in lab.items():
    print(f"{l:22s} median {np.median(d[:, :, b] - d[:, :, a]):8.0f}")
print(f"{'topk->next loop':22s} median {np.median(d[1:, :, 0] - d[:-1, :, 7]):8.0f}")
# CW: gap between consecutive slot services
cw = np.sort(d[:, :, 1].reshape(-1))
print("CW service interval median", np.median(np.diff(cw)), " CW busy (woke->issued) median", np.median(d[:, :, 2] - d[:, :, 1]))
