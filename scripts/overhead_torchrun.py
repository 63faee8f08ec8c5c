#!/usr/bin/env python3
"""Per-step fixed cost of the multi-GPU path, measured under
torchrun with CUDA events per phase: K1 on the rank's shard (records, grid merge
fused in), the NCCL all_gather of W x k records, K2 over W x k records.

    python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 \\
        --master-addr 127.0.0.1 --master-port 29555 scripts/overhead_torchrun.py

Rows: the full cfg2 / cfg5 sweeps and a tiny shard (one tile per CTA slot), so
fixed cost = the tiny step's phases; it is compared with the cfg5 shard time at
N = 1, 2, 4, 8 ranks (0.43 s / N).  Prints one JSON line per row (rank 0)."""

import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_14011_b200 as pk  # noqa: E402
import workloads  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = torch.device(f"cuda:{local}")
    rows = []
    for wl_name, n_override in (("cfg2", None), ("cfg5", None), ("cfg5", 148 * 4 * 128), ("cfg2", 148 * 4 * 128)):
        wl = workloads.WORKLOADS[wl_name]
        vl = workloads.space(wl.space)
        model = workloads.load_model(wl.weights)
        h = pk.Surrogate(local).load(model, wl.precision)
        k = wl.k
        n_space = 1
        for v in vl:
            n_space *= len(v)
        n = n_override or n_space
        from paper_2306_14011_b200.dist import shard_range
        lo, hi = shard_range(n, world, rank)
        desc = pk.SpaceDesc(vl, lo, hi)
        recs = torch.empty((k, 2), dtype=torch.int64, device=dev)
        gathered = torch.empty((world * k, 2), dtype=torch.int64, device=dev)
        idx = torch.empty(k, dtype=torch.int64, device=dev)
        tt = torch.empty(k, dtype=torch.float32, device=dev)
        steps = 5 if n_override is None else 50
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
        for it in range(3 + steps):
            dist.barrier()
            torch.cuda.synchronize()
            e = ev[it - 3] if it >= 3 else None
            if e: e[0].record()
            h.sweep_records_into(desc, k, recs)
            if e: e[1].record()
            dist.all_gather_into_tensor(gathered, recs)
            if e: e[2].record()
            h.merge_topk_into(gathered, world, k, k, idx, tt)
            if e: e[3].record()
        torch.cuda.synchronize()
        ph = [sorted(x[i].elapsed_time(x[i + 1]) * 1e3 for x in ev)[steps // 2] for i in range(3)]
        tot = sorted(x[0].elapsed_time(x[3]) * 1e3 for x in ev)[steps // 2]
        row = {"workload": wl_name, "configs": n, "world": world, "k": k,
               "k1_us": ph[0], "allgather_us": ph[1], "k2_us": ph[2], "step_us": tot}
        if rank == 0:
            print(json.dumps(row), flush=True)
        rows.append(row)
        h.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
