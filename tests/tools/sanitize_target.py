"""Small launches of every kernel family for compute-sanitizer (tests/test_gpu_sanitizer.py).

Run as a script under `compute-sanitizer --tool <memcheck|synccheck|racecheck>`:
the 4-slot 16-bit kernel (sweep, dense, predict), the 3xFP16 and 3xTF32
FP32-path kernels, the general kernel (3 hidden layers), the CTA-pair kernel
(H = 256), an ensemble, and the merge kernel, each on a range of a few tiles
with a ragged tail.  Prints one line per case; correctness is the parity
suite's job, this only exercises the memory / barrier traffic."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_14011_b200 as pk  # noqa: E402
import workloads  # noqa: E402


def main():
    vl2 = workloads.space("cfg2")
    vl3 = workloads.space("cfg3")
    b, n = 1_000_003, 2 * 148 * 128 + 77  # ragged: a partial tile per CTA set
    cases = [
        ("fp16 4-slot", vl2, workloads.load_model("cfg2_14-128-128-1"), "fp16"),
        ("bf16 4-slot", vl2, workloads.load_model("cfg2_14-128-128-1"), "bf16"),
        ("fp32 3xFP16", vl2, workloads.load_model("cfg2_14-128-128-1"), "fp32"),
        ("fp32 3xTF32", vl2, workloads.load_model("cfg2_14-128-128-1"), "fp32_3xtf32"),
        ("tf32 general", vl2, workloads.load_model("cfg2_14-128-128-1"), "tf32"),
        ("fp16 general 3 hidden", vl2, workloads.random_net(vl2, [64, 64, 64], seed=3), "fp16"),
        ("fp16 pair H=256", vl3, workloads.random_net(vl3, [256, 256], seed=4), "fp16"),
        ("fp16 ensemble x3", vl2, workloads.random_net(vl2, [128, 128], seed=5, ensemble=3), "fp16"),
    ]
    for name, vl, model, prec in cases:
        h = pk.Surrogate(0).load(model, prec)
        idx, t, cnt = h.sweep(vl, 32, b, b + n)
        dense = h.eval_range(vl, b, b + 999)
        X = torch.tensor(np.asarray(workloads.predict_rows(vl, 777, seed=1), np.float32), device="cuda:0")
        tp = h.predict(X)
        recs = torch.cat([h.sweep_records(vl, 16, b, b + 5000), h.sweep_records(vl, 16, b + 5000, b + 9000)])
        mi, mt, _ = h.merge_topk(recs, 2, 16, 16)
        torch.cuda.synchronize()
        print(f"{name}: top-1 {int(idx[0])} {float(t[0]):.5f}, dense {float(dense.sum()):.3f}, "
              f"predict {float(tp.sum()):.3f}, merged {int(mi[0])}", flush=True)
    # GPU training (one member: DSMEM pull exchange; two members: push exchange)
    Xs, ys = workloads.training_rows(vl2, 420, seed=2)
    for E in (1, 2):
        inits = [workloads.glorot_init([14, 32, 32, 1], seed=10 + e) for e in range(E)]
        perms = np.stack([workloads.epoch_permutations(420, 2, seed=20 + e) for e in range(E)])
        res = pk.train_ensemble(inits, Xs, ys, perms, dict(max_epochs=2))
        print(f"train E={E}: loss {res[0][2][-1]:.5f}", flush=True)
    print("sanitize_target done")


if __name__ == "__main__":
    main()
