#!/usr/bin/env python3
"""Quick GPU timing probe of the sweep kernel (development aid, not the bench)."""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_14011_b200 as pk  # noqa: E402
import workloads  # noqa: E402

FLOP = {"cfg2": 2 * (14 * 128 + 128 * 128 + 128), "cfg5": 2 * (14 * 128 + 128 * 128 + 128),
        "tiny": 2 * (14 * 32 + 32 * 32 + 32)}


def main():
    names = sys.argv[1:] or ["cfg2"]
    for name in names:
        wl = workloads.WORKLOADS[name]
        vl = workloads.space(wl.space)
        model = workloads.load_model(wl.weights)
        N = int(np.prod([len(v) for v in vl]))
        for prec in ["bf16", "tf32", "fp32"]:
            h = pk.Surrogate(0).load(model, prec)
            desc = pk.SpaceDesc(vl)
            idx = torch.empty(wl.k, dtype=torch.int64, device="cuda")
            t = torch.empty(wl.k, dtype=torch.float32, device="cuda")
            for _ in range(3):
                h.sweep_into(desc, wl.k, idx, t)
            torch.cuda.synchronize()
            h.kernel_timing(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 5
            e0.record()
            for _ in range(reps):
                h.sweep_into(desc, wl.k, idx, t)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            kms, kn = h.kernel_timing_get()
            h.kernel_timing(False)
            kms /= max(kn, 1)
            print(f"{name} {prec}: step {ms:.3f} ms, K1 {kms:.3f} ms, {N / ms * 1e3:.3e} evals/s, "
                  f"{FLOP.get(name, 0) * N / kms / 1e9:.1f} TFLOP/s algorithmic; top1 {int(idx[0])} {float(t[0]):.5f}",
                  flush=True)
            h.close()


if __name__ == "__main__":
    main()
