"""The product multi-GPU path (paper_2306_14011_b200.dist.sweep: CUDA K1 records
on each rank's a1 shard -> one all_gather -> CUDA K2 merge) with W = 2 and 3
ranks sharing the one B200 of the test box, exchanging over a gloo group with
host-staged records.  The merged top-k must be bitwise equal to the W = 1
sweep on every rank (SURVEY §4 derived pin 4, §8(e)); nothing here substitutes
the oracle for the sweep or the merge.  (NCCL needs one GPU per rank: the
driver's SCALE run covers it.)"""

import os
import socket

import numpy as np
import pytest

from tests.helpers import need_gpu

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, weights, prec, k, out_q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2306_14011_b200 as pk
        import workloads
        from paper_2306_14011_b200 import dist as pdist
        vl = workloads.space(name)
        h = pk.Surrogate(0).load(workloads.load_model(weights), prec)
        idx, t = pdist.sweep(h, vl, k)
        torch.cuda.synchronize()
        out_q.put((rank, idx.cpu().numpy().tolist(), t.cpu().numpy().view(np.uint32).tolist(), h.last_launches()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name,weights,prec,k", [(2, "cfg2", "cfg2_14-128-128-1", "fp16", 16),
                                                       (3, "cfg2", "cfg2_14-128-128-1", "fp32", 64),
                                                       (2, "tiny", "tiny_14-32-32-1", "fp32", 1)])
def test_product_path_world_gt_1_bitwise_equals_single(world, name, weights, prec, k):
    pk = need_gpu()
    import torch
    import torch.multiprocessing as mp
    import workloads
    vl = workloads.space(name)
    h = pk.Surrogate(0).load(workloads.load_model(weights), prec)
    i1, t1, _ = h.sweep(vl, k)
    torch.cuda.synchronize()
    ref_i = i1.cpu().numpy().tolist()
    ref_t = t1.cpu().numpy().view(np.uint32).tolist()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, weights, prec, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, gi, gt, launches in got:
        assert gi == ref_i, f"rank {rank}: indices differ from the W = 1 sweep"
        assert gt == ref_t, f"rank {rank}: times differ bitwise from the W = 1 sweep"
        assert launches >= 1  # the last call (the K2 merge of W x k records) ran on the GPU
