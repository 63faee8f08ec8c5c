"""Multi-GPU sweep: index-range shards + ONE all_gather of the per-rank top-k.

SURVEY §8(a) a1 / a10, §8(e): rank r of W sweeps the contiguous shard
[lo_r, hi_r) with q = N // W, rem = N % W, lo_r = r q + min(r, rem) (no u64
overflow of r N); its k best are kept as surr_record rows (idx, key) with
sentinels padding short shards; one ``all_gather_into_tensor`` over NCCL
(NVLink / NVSwitch) collects the W * k records on every rank; the merge kernel
(K2) reduces them to the k best.  Every rank ends with the same, bitwise
identical result, independent of W (the (t, idx) order is total).

One process per GPU (torchrun); ``torch.distributed`` is plumbing only.
"""

from __future__ import annotations

from contextlib import contextmanager

import torch
import torch.distributed as dist


@contextmanager
def nvtx(name: str):
    """NVTX range (sweep / allgather / merge) for nsys timelines; no-op without CUDA."""
    on = torch.cuda.is_available()
    if on:
        torch.cuda.nvtx.range_push(name)
    try:
        yield
    finally:
        if on:
            torch.cuda.nvtx.range_pop()


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    q, rem = divmod(int(n), int(world))
    lo = rank * q + min(rank, rem)
    return lo, lo + q + (1 if rank < rem else 0)


def gather_records(recs: torch.Tensor, group=None) -> torch.Tensor:
    """All ranks' [k, 2] int64 record blocks -> [W * k, 2] in rank order (one collective).

    NCCL exchanges the device tensors directly (NVLink / NVSwitch).  A gloo
    group (several ranks sharing one GPU, or CPU tests) exchanges host copies:
    the records are staged to host memory, gathered, and copied back to the
    device the caller's merge kernel reads; the result is the same bytes."""
    world = dist.get_world_size(group)
    host_staged = recs.is_cuda and dist.get_backend(group) == "gloo"
    src = recs.contiguous().cpu() if host_staged else recs.contiguous()
    out = torch.empty((world * src.shape[0], src.shape[1]), dtype=src.dtype, device=src.device)
    with nvtx("surrogate.allgather"):
        dist.all_gather_into_tensor(out, src, group=group)
    return out.to(recs.device) if host_staged else out


def sweep_distributed(local_sweep, merge, n: int, k: int, group=None):
    """Generic driver: ``local_sweep(lo, hi, k) -> [k, 2] records`` (sorted, sentinel
    padded), ``merge(records [W*k, 2], W, k) -> result``.  Returns merge's result."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(n, world, rank)
    with nvtx("surrogate.sweep_shard"):
        recs = local_sweep(lo, hi, k)
    gathered = gather_records(recs, group)
    with nvtx("surrogate.merge"):
        return merge(gathered, world, k)


def sweep(surrogate, value_lists, k: int, group=None):
    """The product path: K1+K2 on this rank's shard, all_gather, K2 merge.
    Returns (idx int64 [k], t float32 [k]) on every rank."""
    import numpy as np
    n = int(np.prod([len(v) for v in value_lists], dtype=object))

    def local(lo, hi, kk):
        return surrogate.sweep_records(value_lists, kk, lo, hi)

    def merge(recs, world, kk):
        idx, t, _ = surrogate.merge_topk(recs, world, kk, kk)
        return idx, t

    return sweep_distributed(local, merge, n, k, group)


def sweep_campaign(make_campaign, merge, n: int, k: int, group=None):
    """Checkpointed multi-GPU sweep: each rank runs
    ``make_campaign(lo, hi)`` (a `campaign.Campaign` over its shard, with its
    own checkpoint file) to completion, then the per-rank records are exchanged
    with one all_gather and merged as in `sweep_distributed`."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(n, world, rank)
    recs = make_campaign(lo, hi).run()
    return merge(gather_records(recs, group), world, k)


def campaign(surrogate, value_lists, k: int, chunk: int, ckpt_dir: str | None = None, tag: str = "",
             every: int = 1, group=None):
    """The product path of a checkpointed full-space sweep on every rank:
    chunks of K1 + K2, K2 folds, per-rank checkpoint ``ckpt_dir/rank<r>.npz``,
    one all_gather, K2 merge.  Returns (idx int64 [k], t float32 [k])."""
    import os

    import numpy as np

    from . import campaign as cp
    n = int(np.prod([len(v) for v in value_lists], dtype=object))
    rank = dist.get_rank(group)

    def make(lo, hi):
        path = os.path.join(ckpt_dir, f"rank{rank}.npz") if ckpt_dir else None
        return cp.for_surrogate(surrogate, value_lists, k, lo, hi, chunk, path, every, tag)

    def merge(recs, world, kk):
        idx, t, _ = surrogate.merge_topk(recs, world, kk, kk)
        return idx, t

    return sweep_campaign(make, merge, n, k, group)
