"""Multi-process (world size 2, gloo, CPU) coverage of the N > 1 path's host
logic: shard bounds, the record exchange (one all_gather) and the merge.  The
per-rank sweep and the merge are the oracle's here (the CUDA kernels need a
B200); the plumbing is the product's paper_2306_14011_b200.dist."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_14011_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _keys(t):
    u = np.asarray(t, np.float32).view(np.uint32)
    return np.where(np.isnan(t), 0xFFFFFFFF, np.where(u & 0x80000000, ~u, u | 0x80000000)).astype(np.uint32)


def _records(idx, t, k):
    """[k, 2] int64 rows (idx, key) padded with sentinels, like surr_record."""
    out = np.zeros((k, 2), np.int64)
    out[:, 0] = -1
    out[:, 1] = 0xFFFFFFFF
    n = len(idx)
    out[:n, 0] = np.asarray(idx, np.uint64).view(np.int64)
    out[:n, 1] = _keys(t).astype(np.int64)
    return torch.from_numpy(out)


def _worker(rank, world, port, n_range, k, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import workloads
    from oracle import sweep as osweep
    vl = workloads.space("cfg2")
    model = workloads.random_net(vl, [8, 8], seed=4)
    base = 50_000_000

    def local(lo, hi, kk):
        i, t = osweep.topk(model, vl, kk, base + lo, base + hi) if hi > lo else (np.zeros(0, np.uint64), np.zeros(0))
        return _records(i, t.astype(np.float32), kk)

    def merge(recs, w, kk):
        r = recs.numpy()
        valid = r[:, 0] != -1
        keys = r[valid, 1].astype(np.uint64)
        idx = r[valid, 0].astype(np.uint64)
        o = np.lexsort((idx, keys))[:kk]
        return idx[o], keys[o], recs.shape[0]

    res = pdist.sweep_distributed(local, merge, n_range, k)
    out_q.put((rank, res[0].tolist(), res[1].tolist(), res[2], pdist.shard_range(n_range, world, rank)))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_range,k", [(60_001, 12), (5, 8)])
def test_two_rank_sweep_matches_single_process(n_range, k):
    import workloads
    from oracle import sweep as osweep
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_range, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort()
    # every rank ends with the identical merged result
    assert got[0][1:3] == got[1][1:3]
    assert got[0][3] == world * k          # one all_gather of k records per rank
    assert got[0][4] == (0, (n_range + 1) // 2) and got[1][4][1] == n_range
    vl = workloads.space("cfg2")
    model = workloads.random_net(vl, [8, 8], seed=4)
    ri, rt = osweep.topk(model, vl, k, 50_000_000, 50_000_000 + n_range)
    assert got[0][1] == [int(i) for i in ri]
    assert got[0][2] == [int(x) for x in _keys(rt.astype(np.float32))]


def test_shard_range_properties():
    for n in [0, 1, 7, 170859375, 2 ** 63 + 5]:
        for w in [1, 2, 3, 8]:
            parts = [pdist.shard_range(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        pdist.shard_range(10, 2, 2)
