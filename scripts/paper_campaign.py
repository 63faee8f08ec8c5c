#!/usr/bin/env python3
"""The paper's whole search space (10^7 x 12^7 = 3.58e14 configs)
swept to its top-1024 on one B200 as a checkpointed campaign (SURVEY 8(f)
NEXT-2; `paper_2306_14011_b200.campaign`), across as many GPU calls as it
takes.

    python scripts/paper_campaign.py --ckpt campaign/paper_fp16.npz --budget-s 3300

Each call resumes from the checkpoint, sweeps chunks of 2^38 configs (K1 with
the fused CTA merge tree, then K2 folds the chunk's records into the running
top-k, all on the device) until the time budget is spent, checkpoints after
every chunk and appends one line per call to <ckpt>.log.jsonl (chunks,
configs, CUDA-event device time, wall time).  When the range is finished it
writes <ckpt>.result.json: the top-1024 (index, decoded parameter values, t),
the total device time and rate, and a check of the returned configs against
the float64 oracle evaluated at those indices (the completeness of an
exhaustive 3.58e14 sweep cannot be enumerated on the CPU; windows of the same
space are checked exhaustively by tests/test_gpu_parity.py)."""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2306_14011_b200 as pk  # noqa: E402
import workloads  # noqa: E402
from paper_2306_14011_b200 import campaign as cp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ckpt", default=os.path.join(ROOT, "campaign", "paper_fp16.npz"))
    ap.add_argument("--budget-s", type=float, default=3300.0)
    ap.add_argument("--chunk-log2", type=int, default=38)
    ap.add_argument("--precision", default="fp16")
    ap.add_argument("--end", type=int, default=0, help="stop at this index (0: the whole space; tests)")
    a = ap.parse_args()
    wl = workloads.WORKLOADS["paper"]
    vl = workloads.space(wl.space)
    model = workloads.load_model(wl.weights)
    radix = [len(v) for v in vl]
    N = int(np.prod(radix, dtype=object))
    end = a.end or N
    os.makedirs(os.path.dirname(os.path.abspath(a.ckpt)), exist_ok=True)
    h = pk.Surrogate(0).load(model, a.precision)
    camp = cp.for_surrogate(h, vl, wl.k, 0, end, 1 << a.chunk_log2, path=a.ckpt, every=1,
                            tag=f"paper {a.precision}")
    start_next = camp.next
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dev_ms, n = 0.0, 0
    t0 = time.time()
    log = open(a.ckpt + ".chunks.jsonl", "a")  # one line per chunk (survives a killed call)
    while not camp.finished and time.time() - t0 < a.budget_s:
        lo = camp.next
        ev0.record()
        camp.step()  # the chunk's sweep + fold, then the checkpoint write (host)
        ev1.record()
        ev1.synchronize()
        ms = ev0.elapsed_time(ev1)
        dev_ms += ms
        n += 1
        log.write(json.dumps({"lo": lo, "hi": camp.next, "device_ms": ms}) + "\n")
        log.flush()
    log.close()
    wall = time.time() - t0
    line = {"call_start": t0, "chunks": n, "from": start_next, "to": camp.next, "configs": camp.next - start_next,
            "device_s": dev_ms / 1e3, "wall_s": wall, "finished": camp.finished, "end": end,
            "precision": a.precision, "gpu": torch.cuda.get_device_name(0)}
    with open(a.ckpt + ".log.jsonl", "a") as f:
        f.write(json.dumps(line) + "\n")
    print(json.dumps(line), flush=True)
    if not camp.finished:
        return
    calls = [json.loads(x) for x in open(a.ckpt + ".log.jsonl")]
    recs = camp.recs.cpu().numpy()
    count = min(wl.k, end)
    idx, t = cp.records_to_result(recs, count)
    from oracle import space as osp, sweep as osweep  # verification of the returned configs only
    digits = osp.decode(idx.astype(np.uint64), radix)
    vals = osp.values_of(digits, vl)
    t_ref = osweep.times_at(model, vl, idx.astype(np.uint64))
    den = np.maximum(np.abs(t_ref), 1e-3 * model["y_scale"])
    rel = np.abs(t.astype(np.float64) - t_ref) / den
    # device time and configs from the per-chunk log (calls killed by a time
    # limit leave no call line; chunks swept before the log existed count as
    # untimed)
    chunks = [json.loads(x) for x in open(a.ckpt + ".chunks.jsonl")]
    configs = sum(c["hi"] - c["lo"] for c in chunks)
    dev_s = sum(c["device_ms"] for c in chunks) / 1e3
    out = {"space": f"paper: 10^7 x 12^7 = {N} configs (PAPER.md:241)", "range": [0, end], "k": wl.k,
           "precision": a.precision, "net": "-".join(map(str, model["widths"])), "weights": wl.weights,
           "calls_logged": len(calls), "configs_timed": configs, "device_s_timed": dev_s,
           "evals_per_s": configs / dev_s, "configs_untimed": end - configs,
           "chunk": 1 << a.chunk_log2,
           "sorted": bool(np.all(np.diff(t) >= 0)), "unique": int(len(np.unique(idx))) == count,
           "oracle_max_rel_err_at_returned": float(rel.max()),
           "top": [{"idx": int(i), "t": float(tt), "t_oracle": float(tr), "values": [int(x) for x in v]}
                   for i, tt, tr, v in zip(idx[:64], t[:64], t_ref[:64], vals[:64])],
           "all_idx": [int(i) for i in idx], "all_t": [float(x) for x in t]}
    with open(a.ckpt + ".result.json", "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("configs_timed", "device_s_timed", "evals_per_s", "sorted", "unique",
                                          "oracle_max_rel_err_at_returned")}), flush=True)


if __name__ == "__main__":
    main()
