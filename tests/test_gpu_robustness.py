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


@pytest.mark.parametrize("name,weights,prec,k,begin,end", [
    ("cfg2", "cfg2_14-128-128-1", "fp16", 16, 0, None),
    ("cfg5", "cfg5_14-128-128-1", "fp16", 1024, 5_000_000_000, 5_000_000_000 + (1 << 27) + 77),
    ("cfg2", "cfg2_14-128-128-1", "fp32", 64, 1000, 1000 + (1 << 24)),
    ("cfg3", "cfg3_14-256-256-256-1", "fp16", 64, 0, 1 << 24),
    ("cfg2", "cfg4_17-128-128-1_x8", "fp16", 16, 0, 1 << 22),
    ("tiny", "tiny_14-32-32-1", "fp32", 1, 0, None),
    ("cfg2", "cfg2_14-128-128-1", "fp16", 1024, 0, 3000),   # fewer configs than a full grid of lists
    # odd and tiny grids of the merge tree (4 tiles of 128 rows per CTA): 37, 3, 2, 1 CTAs
    ("cfg2", "cfg2_14-128-128-1", "fp16", 64, 0, 512 * 37 - 5),
    ("cfg2", "cfg2_14-128-128-1", "fp16", 1024, 10, 10 + 512 * 3),
    ("cfg2", "cfg2_14-128-128-1", "bf16", 7, 99, 99 + 512 * 2),
    ("cfg2", "cfg2_14-128-128-1", "fp16", 5, 123, 123 + 300),
    ("cfg5", "cfg5_14-128-128-1", "fp16", 1000, 7, 7 + 512 * 147 + 1),  # 148 CTAs, the last one a single row
])
def test_fused_grid_merge_equals_k2(pk, monkeypatch, name, weights, prec, k, begin, end):
    """a9 in K1 (a binary tree of CTAs merges the grid's lists) == K1 + the
    separate K2 merge, bitwise, and the sweep is one kernel launch; odd grids
    (nodes without a sibling), a grid of one and repeated launches (tickets
    re-armed) included."""
    import torch
    vl = workloads.space(name)
    model = workloads.load_model(weights)
    if model["const_features"].size or "cfg4" in weights:
        model = workloads.with_device(model, workloads.device_features("onehot", "V100"))
    h = pk.Surrogate(0).load(model, prec)
    N = int(np.prod([len(v) for v in vl], dtype=object))
    end = N if end is None else end
    i1, t1, c1 = h.sweep(vl, k, begin, end)
    torch.cuda.synchronize()
    n1 = h.last_launches()
    monkeypatch.setenv("SURR_NO_FUSED_MERGE", "1")
    i2, t2, c2 = h.sweep(vl, k, begin, end)
    torch.cuda.synchronize()
    n2 = h.last_launches()
    assert c1 == c2 == min(k, end - begin)
    assert torch.equal(i1, i2) and torch.equal(t1.view(torch.int32), t2.view(torch.int32))
    members = len(model["members"])
    if members == 8:  # the single-pass ensemble (CTA pairs): one launch either way
        assert n1 == 1 and n2 == 2
    else:
        assert n1 == members and n2 == members + 1  # fused: K1 only
    # repeated fused sweeps re-arm the ticket
    monkeypatch.delenv("SURR_NO_FUSED_MERGE")
    for _ in range(3):
        i3, t3, _ = h.sweep(vl, k, begin, end)
    torch.cuda.synchronize()
    assert torch.equal(i1, i3)


@pytest.mark.parametrize("members,prec,begin,n", [(8, "fp16", 0, None), (8, "bf16", 77_777_777, (1 << 20) + 13),
                                                  (4, "fp16", 170859375 - 300_001, 300_001),
                                                  (8, "fp16", 5, 1000)])
def test_single_pass_ensemble_equals_multipass(pk, monkeypatch, members, prec, begin, n):
    """the E-member ensemble in one pass on CTA pairs (members
    split, per-row predictions exchanged through distributed shared memory, no
    HBM accumulator) is bitwise the multi-pass path (one K1 pass per member with
    an fp32 accumulator, members summed in order e = 0 .. E-1), dense times and
    top-k, in one kernel launch per sweep."""
    import torch
    vl = workloads.space("cfg2")
    if members == 8:
        model = workloads.with_device(workloads.load_model("cfg4_17-128-128-1_x8"),
                                      workloads.device_features("onehot", "P100"))
    else:
        model = workloads.random_net(vl, [128, 128], seed=31, ensemble=members)
    h = pk.Surrogate(0).load(model, prec)
    N = 170859375
    end = N if n is None else begin + n
    k = 16
    i1, t1, _ = h.sweep(vl, k, begin, end)
    torch.cuda.synchronize()
    assert h.last_launches() == 1
    d1 = h.eval_range(vl, begin, min(end, begin + (1 << 20)))
    torch.cuda.synchronize()
    monkeypatch.setenv("SURR_NO_ENS_PAIR", "1")
    i2, t2, _ = h.sweep(vl, k, begin, end)
    torch.cuda.synchronize()
    assert h.last_launches() == members  # multi-pass: one K1 per member (merge fused into the last)
    d2 = h.eval_range(vl, begin, min(end, begin + (1 << 20)))
    torch.cuda.synchronize()
    assert torch.equal(d1.view(torch.int32), d2.view(torch.int32)), \
        f"{int((d1 != d2).sum())} rows differ between the single-pass and the multi-pass ensemble"
    assert torch.equal(i1, i2) and torch.equal(t1.view(torch.int32), t2.view(torch.int32))
    # and against the oracle's float64 mean on a slice
    ref = osweep.times(model, vl, begin, begin + min(4096, end - begin))
    assert rel_err(d1[:len(ref)].cpu().numpy(), ref, model["y_scale"]).max() <= TOL[prec]
