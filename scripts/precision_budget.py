#!/usr/bin/env python3
"""Emulate the kernel's rounding points in numpy to size the BF16 / FP32-path error.

A development study, not part of any test: it
models where the CUDA path rounds (LUT z -> bf16 or tf32 hi/lo, weights ->
bf16 or tf32 hi/lo, fp32 accumulation, hidden activations -> bf16) and
compares t against float64, using rel = |dt| / max(|t|, 1e-3 sigma_y) (G16).

    python scripts/precision_budget.py cfg2 [n]
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import workloads  # noqa: E402


def bf16(x):
    a = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((a + 0x7FFF + ((a >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def tf32(x):
    a = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((a + 0xFFF + ((a >> 13) & 1)) >> 13) << 13   # round-to-nearest into 10-bit mantissa
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def f32(x):
    return np.asarray(x, np.float32).astype(np.float64)


def fp16(x):
    return np.asarray(x, np.float32).astype(np.float16).astype(np.float64)


def split_fp16(x):
    hi = fp16(x)
    lo = fp16(f32(x) - hi)
    return hi, lo


def split_tf32(x):
    hi = tf32(x)
    lo = tf32(f32(x) - hi)
    return hi, lo


def emulate(model, Z, mode, l1="bf16"):
    m = model["members"][0]
    W, b = m["W"], m["b"]
    L = len(W)
    h = f32(Z)
    for l in range(L - 1):
        if mode == "bf16":
            if l == 0 and l1 == "bf16x3":
                zh = bf16(h); zl = bf16(h - zh)
                wh = bf16(W[0]); wl = bf16(f32(W[0]) - wh)
                d = f32(zh @ wh + zl @ wh + zh @ wl + (bf16(b[0]) + bf16(f32(b[0]) - bf16(b[0]))))
            elif l == 0:
                d = f32(bf16(h) @ bf16(W[0]) + bf16(b[0]))
            else:
                d = f32(f32(bf16(h) @ bf16(W[l])) + f32(b[l]))
        elif mode == "fp16":
            d = f32(f32(fp16(h) @ fp16(W[l])) + (fp16(b[l]) if l == 0 else f32(b[l])))
        elif mode == "fp16x3":
            hh, hl = split_fp16(h)
            wh, wl = split_fp16(W[l])
            if l == 0:
                bh, bl = split_fp16(b[0])
                d = f32(hh @ wh + hh @ wl + hl @ wh + bh + bl)
            else:
                d = f32(f32(hh @ wh + hh @ wl + hl @ wh) + f32(b[l]))
        else:
            hh, hl = split_tf32(h)
            wh, wl = split_tf32(W[l])
            if l == 0:
                bh, bl = split_tf32(b[0])
                d = f32(hh @ wh + hh @ wl + hl @ wh + bh + bl)
            else:
                d = f32(f32(hh @ wh + hh @ wl + hl @ wh) + f32(b[l]))
        h = np.maximum(d, 0.0)
    y = f32(h @ f32(W[-1]) + f32(b[-1]))[:, 0]
    return f32(model["y_mean"] + model["y_scale"] * y)


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 400000
    wl = workloads.WORKLOADS[name]
    vl = workloads.space(wl.space)
    model = workloads.load_model(wl.weights)
    rng = np.random.default_rng(1)
    N = oracle.space.cardinality([len(v) for v in vl])
    idx = np.unique(rng.integers(0, N, n, dtype=np.uint64))
    X = oracle.space.values_of(oracle.space.decode(idx, [len(v) for v in vl]), vl)
    Z = (X - model["x_shift"]) / model["x_scale"]
    t = oracle.sweep.times_at(model, vl, idx)
    den = np.maximum(np.abs(t), 1e-3 * model["y_scale"])
    for mode, l1 in [("bf16", "bf16"), ("bf16", "bf16x3"), ("fp16", None), ("fp16x3", None), ("fp32", None)]:
        te = emulate(model, Z, mode, l1)
        rel = np.abs(te - t) / den
        print(f"{name} {mode:5s} l1={l1}: max {rel.max():.3e}  p99.9 {np.quantile(rel, 0.999):.3e}"
              f"  median {np.median(rel):.3e}  t in [{t.min():.3f},{t.max():.3f}]")


if __name__ == "__main__":
    main()
