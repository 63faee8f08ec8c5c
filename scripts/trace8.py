#!/usr/bin/env python3
"""CTA 0 timeline of the pipelined K1 (sweep_kernel8, -DSURR_TRACE build).
Events per (round, slot): 0 loop top, 1 woke on D1, 2 L2a issued (epilogue-1
done), 3 L2a-shadow work done (previous tile finished, A0 stored), 4 woke on
D2a, 5 L2b issued + half a done, 6 woke on D2b, 7 next L1 issued + 32 columns."""
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
for j in range(20, 22):
    for s in range(4):
        print(f"round {j} slot {s}: " + " ".join(f"{e}={int(t[j, s, e] - t0)}" for e in range(8) if t[j, s, e] > 0))
d = t[10:50]
per = np.median(np.diff(d[:, 0, 0]))
print("cycles per round (4 tiles):", per, "-> per tile", per / 4, " tensor-bound share", 2560 / per)
names = ["top->wD1", "epi1+issue L2a", "L2a shadow work", "wait D2a", "ldA+L2b+halfA", "wait D2b", "ldB+L1+32col"]
for e in range(7):
    print(f"{names[e]:18s} median {np.median(d[:, :, e + 1] - d[:, :, e]):8.0f}")
print(f"{'loop->top':18s} median {np.median(d[1:, :, 0] - d[:-1, :, 7]):8.0f}")
