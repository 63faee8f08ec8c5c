"""Error behaviour and edge cases of the boundary (include/surrogate.h) found by
the round-1 code review: a rejected space leaves no stale cache, merges with
k > k_in and odd list counts, digits wider than a byte, non-finite weights, a
diverging fit, campaign checkpoints bound to the loaded model, and table /
weight replacement while earlier sweeps are still queued."""

import numpy as np
import pytest

import workloads
from oracle import sweep as osweep
from tests.helpers import TOL, need_gpu, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    return need_gpu()


def test_rejected_space_leaves_no_stale_cache(pk):
    import torch
    vl = workloads.space("cfg2")
    h = pk.Surrogate(0).load(workloads.load_model("cfg2_14-128-128-1"), "bf16")
    i0, t0, _ = h.sweep(vl, 16, 0, 1 << 20)
    torch.cuda.synchronize()
    # a space whose value table cannot fit (9e8 entries in the first pair group)
    big = [list(range(1, 30001)), list(range(1, 30001))] + [[5]] * 12
    with pytest.raises(pk.SurrogateError, match="too large"):
        h.sweep(big, 16, 0, 1 << 20)
    # the previous space again: rebuilt from its descriptor, identical result
    i1, t1, _ = h.sweep(vl, 16, 0, 1 << 20)
    torch.cuda.synchronize()
    assert torch.equal(i0, i1) and torch.equal(t0, t1)


@pytest.mark.parametrize("lists,k_in,k", [(4, 4, 16), (5, 3, 16), (3, 16, 4), (7, 1, 5), (1, 8, 20)])
def test_merge_k_larger_than_k_in_and_odd_lists(pk, lists, k_in, k):
    import torch
    rng = np.random.default_rng(lists * 100 + k_in)
    recs = []
    for _ in range(lists):
        idx = np.sort(rng.choice(10_000, k_in, replace=False)).astype(np.int64)
        keys = np.sort(rng.integers(0x80000000, 0x90000000, k_in)).astype(np.int64)
        recs.append(np.stack([idx, keys], axis=1))
    flat = np.concatenate(recs)
    h = pk.Surrogate(0).load(workloads.random_net(workloads.space("tiny"), [32, 32], seed=1), "fp16")
    i, t, r = h.merge_topk(torch.from_numpy(flat).cuda(), lists, k_in, k)
    torch.cuda.synchronize()
    o = np.lexsort((flat[:, 0], flat[:, 1]))[:k]
    exp = flat[o]
    got = r.cpu().numpy()
    n = min(k, lists * k_in)
    assert np.array_equal(got[:n, 0], exp[:n, 0]) and np.array_equal(got[:n, 1] & 0xFFFFFFFF, exp[:n, 1])
    assert (got[n:, 0] == -1).all()  # padding: sentinels


def test_decode_radix_above_256_refused(pk):
    vl = [list(range(1, 301)), [1, 2]]
    model = workloads.random_net(vl, [32, 32], seed=2)
    h = pk.Surrogate(0).load(model, "fp32")
    with pytest.raises(pk.SurrogateError, match="256"):
        h.decode_range(vl, 0, 100)


def test_non_finite_weights_refused(pk):
    model = workloads.random_net(workloads.space("tiny"), [32, 32], seed=3)
    model["members"][0]["W"][1][3, 7] = np.nan
    with pytest.raises(pk.SurrogateError, match="non-finite"):
        pk.Surrogate(0).load(model, "fp16")
    model = workloads.random_net(workloads.space("tiny"), [32, 32], seed=3)
    model["members"][0]["b"][0][0] = np.inf
    with pytest.raises(pk.SurrogateError, match="non-finite"):
        pk.Surrogate(0).load(model, "fp32")


def test_diverging_fit_is_an_error(pk):
    vl = workloads.space("cfg2")
    Xs, ys = workloads.training_rows(vl, 800, seed=5)
    W, b = workloads.glorot_init([14, 32, 32, 1], seed=5)
    W0 = [w.copy() for w in W]
    with pytest.raises(pk.SurrogateError, match="non-finite training loss"):
        pk.train(W, b, Xs, ys, hyper=dict(lr0=1e30, max_epochs=5))
    assert all(np.array_equal(a, c) for a, c in zip(W, W0))  # caller's arrays untouched


def test_campaign_checkpoint_bound_to_model(pk, tmp_path):
    from paper_2306_14011_b200 import campaign as cp
    vl = workloads.space("cfg2")
    path = str(tmp_path / "c.npz")
    h = pk.Surrogate(0).load(workloads.load_model("cfg2_14-128-128-1"), "fp16")
    c = cp.for_surrogate(h, vl, 8, 0, 1 << 20, 1 << 18, path)
    c.run(max_chunks=1)
    c.save()
    # same space / range / k / chunk, other weights -> refused
    h2 = pk.Surrogate(0).load(workloads.random_net(vl, [128, 128], seed=9), "fp16")
    with pytest.raises(ValueError, match="another campaign"):
        cp.for_surrogate(h2, vl, 8, 0, 1 << 20, 1 << 18, path)
    # same weights, other precision -> refused
    h3 = pk.Surrogate(0).load(workloads.load_model("cfg2_14-128-128-1"), "bf16")
    with pytest.raises(ValueError, match="another campaign"):
        cp.for_surrogate(h3, vl, 8, 0, 1 << 20, 1 << 18, path)
    # the same model resumes
    c2 = cp.for_surrogate(pk.Surrogate(0).load(workloads.load_model("cfg2_14-128-128-1"), "fp16"), vl, 8, 0,
                          1 << 20, 1 << 18, path)
    assert c2.resumed_from == 1 << 18


def test_table_and_weight_swaps_while_sweeps_are_queued(pk):
    """Many space changes and a weight reload queued back to back on a busy
    stream (no host synchronisation in between): every result must be the one
    of its own space and weights (two-slot upload rings, stream-ordered)."""
    import torch
    spaces = [workloads.space("cfg2"), workloads.space("cfg5"), workloads.space("cfg3")]
    mA = workloads.load_model("cfg2_14-128-128-1")
    mB = workloads.random_net(spaces[0], [128, 128], seed=12)
    h = pk.Surrogate(0).load(mA, "fp32")
    st = torch.cuda.Stream()
    ref = {}
    for si, vl in enumerate(spaces):
        for name, m in (("A", mA), ("B", mB)):
            t = osweep.times(m, vl, 1000, 1000 + 4096)
            ref[(si, name)] = t
    outs = []
    with torch.cuda.stream(st):
        for rep in range(3):
            for name, m in (("A", mA), ("B", mB)):
                if rep or name == "B":
                    h.load(m, "fp32")
                for si, vl in enumerate(spaces):
                    outs.append(((si, name), h.eval_range(vl, 1000, 1000 + 4096, stream=st)))
    torch.cuda.synchronize()
    for key, t in outs:
        assert rel_err(t.cpu().numpy(), ref[key], 0.3).max() <= TOL["fp32"], key
