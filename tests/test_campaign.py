"""Checkpointed chunked sweeps (paper_2306_14011_b200.campaign, SURVEY 8(f)
NEXT-2): host logic on CPU with the oracle as the per-chunk sweep.  A chunked,
interrupted and resumed campaign must return exactly the oracle's one-shot
top-k of the range (the (t, idx) order is total, so the result is unique)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_14011_b200 import campaign as cp
from paper_2306_14011_b200 import dist as pdist

BASE = 40_000_000


def _keys(t):
    u = np.asarray(t, np.float32).view(np.uint32)
    return np.where(u & 0x80000000, ~u, u | 0x80000000).astype(np.uint32)


def _records(idx, t, k):
    out = np.zeros((k, 2), np.int64)
    out[:, 0] = cp.SENTINEL_IDX
    out[:, 1] = cp.SENTINEL_KEY
    n = len(idx)
    out[:n, 0] = np.asarray(idx, np.uint64).view(np.int64)
    out[:n, 1] = _keys(t).astype(np.int64)
    return out


def _oracle_fns():
    import workloads
    from oracle import sweep as osweep
    vl = workloads.space("cfg2")
    model = workloads.random_net(vl, [8, 8], seed=9)

    def local(lo, hi, k):
        if hi <= lo:
            return _records([], [], k)
        i, t = osweep.topk(model, vl, k, BASE + lo, BASE + hi)
        return _records(np.asarray(i, np.uint64) - np.uint64(BASE), np.asarray(t, np.float32), k)

    def merge(recs, lists, k):
        r = np.asarray(recs)
        valid = r[:, 0] != cp.SENTINEL_IDX
        keys, idx = r[valid, 1].astype(np.uint64), r[valid, 0].astype(np.uint64)
        o = np.lexsort((idx, keys))[:k]
        out = _records([], [], k)
        out[:len(o), 0] = idx[o].view(np.int64)
        out[:len(o), 1] = keys[o].astype(np.int64)
        return out

    return local, merge


@pytest.mark.parametrize("n,k,chunk", [(50_000, 16, 7_001), (50_000, 16, 100_000), (9, 16, 4), (30_000, 1, 1_000)])
def test_chunked_equals_one_shot(n, k, chunk):
    local, merge = _oracle_fns()
    got = cp.Campaign(local, merge, k, 0, n, chunk).run()
    np.testing.assert_array_equal(got, local(0, n, k))


def test_interrupt_and_resume(tmp_path):
    local, merge = _oracle_fns()
    path = str(tmp_path / "c.npz")
    n, k, chunk = 40_000, 16, 3_000
    a = cp.Campaign(local, merge, k, 0, n, chunk, path, every=2, fp="x")
    a.run(max_chunks=5)            # checkpoint after chunks 2 and 4
    assert not a.finished and a.next == 15_000
    b = cp.Campaign(local, merge, k, 0, n, chunk, path, every=2, fp="x")
    assert b.resumed_from == 12_000  # the last checkpoint, not the last chunk swept
    got = b.run()
    assert b.finished
    np.testing.assert_array_equal(got, local(0, n, k))
    c = cp.Campaign(local, merge, k, 0, n, chunk, path, every=2, fp="x")  # finished checkpoint: nothing left
    assert c.finished
    np.testing.assert_array_equal(c.run(), got)


def test_checkpoint_of_another_campaign_is_refused(tmp_path):
    local, merge = _oracle_fns()
    path = str(tmp_path / "c.npz")
    cp.Campaign(local, merge, 8, 0, 10_000, 1_000, path, fp="a").run(max_chunks=1)
    with pytest.raises(ValueError):
        cp.Campaign(local, merge, 8, 0, 10_000, 1_000, path, fp="b")
    with pytest.raises(ValueError):
        cp.Campaign(local, merge, 16, 0, 10_000, 1_000, path, fp="a")


def test_empty_range_and_result_conversion():
    local, merge = _oracle_fns()
    recs = cp.Campaign(local, merge, 4, 10, 10, 5).run()
    assert np.all(recs[:, 0] == cp.SENTINEL_IDX)
    r = local(0, 1000, 4)
    idx, t = cp.records_to_result(r, 4)
    assert idx.dtype == np.uint64 and t.dtype == np.float32
    np.testing.assert_array_equal(_keys(t).astype(np.int64), r[:4, 1])


def test_fingerprint_changes_with_every_field():
    vl = [[1, 2], [3, 4, 5]]
    base = cp.fingerprint(vl, 4, 0, 6, "m")
    assert base == cp.fingerprint(vl, 4, 0, 6, "m")
    for other in [cp.fingerprint([[1, 2], [3, 4, 6]], 4, 0, 6, "m"), cp.fingerprint(vl, 5, 0, 6, "m"),
                  cp.fingerprint(vl, 4, 1, 6, "m"), cp.fingerprint(vl, 4, 0, 5, "m"), cp.fingerprint(vl, 4, 0, 6, "n")]:
        assert other != base


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, k, ckpt, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    local, merge = _oracle_fns()

    def make(lo, hi):
        c = cp.Campaign(local, merge, k, lo, hi, 2_500, os.path.join(ckpt, f"rank{rank}.npz"), fp="w2",
                        to_numpy=lambda r: np.asarray(r), from_numpy=lambda a: a)
        if c.resumed_from is None:
            c.run(max_chunks=2)  # first session: interrupted
            c = cp.Campaign(local, merge, k, lo, hi, 2_500, os.path.join(ckpt, f"rank{rank}.npz"), fp="w2",
                            to_numpy=lambda r: np.asarray(r), from_numpy=lambda a: a)
        return _TorchWrap(c)

    def gmerge(recs, w, kk):
        return merge(recs.numpy(), w, kk)

    res = pdist.sweep_campaign(make, gmerge, n, k)
    out_q.put((rank, res.tolist()))
    dist.destroy_process_group()


class _TorchWrap:  # the gloo all_gather wants torch tensors
    def __init__(self, c):
        self.c = c

    def run(self):
        return torch.from_numpy(np.ascontiguousarray(self.c.run()))


def test_two_rank_checkpointed_campaign(tmp_path):
    n, k, world = 23_457, 12, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, k, str(tmp_path), q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    local, _ = _oracle_fns()
    ref = local(0, n, k).tolist()
    assert got[0] == ref and got[1] == ref
