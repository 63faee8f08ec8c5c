"""GPU path (through the C ABI) against the CPU oracle on the same seeded inputs.

Sizes: the tiny space in full; cfg2 (15^7) on ragged sub-ranges spanning many
tiles; full-size sweeps checked by re-evaluating every returned item with the
oracle and by the closed-form pins (all-ties net, affine net).
"""

import numpy as np
import pytest
import torch

import workloads
from oracle import space as ospace
from oracle import sweep as osweep
from tests import pins
from tests.helpers import TOL, check_topk, need_gpu, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pk():
    return need_gpu()


def _handle(pk, model, prec):
    return pk.Surrogate(0).load(model, prec)


# ------------------------------------------------------------------ decode (a2)
@pytest.mark.parametrize("name,first,n", [("tiny", 0, 2 ** 14), ("cfg2", 0, 1 << 16),
                                          ("cfg2", 170859375 - 5000, 5000), ("cfg5", 13492928512 - 70000, 70000),
                                          ("cfg5", 7_000_000_123, 100000), ("paper", 358318080000000 - 4096, 4096),
                                          ("paper", 123456789012345, 65536)])
def test_decode_bit_exact(pk, name, first, n):
    vl = workloads.space(name)
    model = workloads.random_net(vl, [32, 32], seed=1)
    h = _handle(pk, model, "bf16")
    got = h.decode_range(vl, first, n).cpu().numpy().astype(np.int64)
    ref = ospace.decode(np.arange(first, first + n, dtype=np.uint64), workloads.radices(name))
    assert np.array_equal(got, ref)


# ------------------------------------------------------------------ dense t(I)
@pytest.mark.parametrize("prec", ["fp32", "fp32_3xtf32", "tf32", "fp16", "bf16"])
def test_tiny_all_times(pk, prec):
    vl = workloads.space("tiny")
    model = workloads.load_model("tiny_14-32-32-1")
    h = _handle(pk, model, prec)
    t = h.eval_range(vl, 0, 2 ** 14).cpu().numpy()
    ref = osweep.times(model, vl, 0, 2 ** 14)
    e = rel_err(t, ref, model["y_scale"])
    assert e.max() <= TOL[prec], f"{prec}: max rel err {e.max():.3e}"


@pytest.mark.parametrize("prec", ["fp32", "fp32_3xtf32", "tf32", "fp16", "bf16"])
@pytest.mark.parametrize("begin,n", [(0, 1 << 18), (98_765_431, (1 << 18) + 77), (170859375 - 100003, 100003)])
def test_cfg2_slice_times(pk, prec, begin, n):
    vl = workloads.space("cfg2")
    model = workloads.load_model("cfg2_14-128-128-1")
    h = _handle(pk, model, prec)
    t = h.eval_range(vl, begin, begin + n).cpu().numpy()
    ref = osweep.times(model, vl, begin, begin + n)
    e = rel_err(t, ref, model["y_scale"])
    assert e.max() <= TOL[prec], f"{prec}: max rel err {e.max():.3e} at {begin + int(np.argmax(e))}"


def test_predict_matches_oracle_and_sweep_bitwise(pk):
    vl = workloads.space("cfg2")
    model = workloads.load_model("cfg2_14-128-128-1")
    for prec in ["bf16", "fp16", "fp32", "fp32_3xtf32"]:
        h = _handle(pk, model, prec)
        # rows = configs [b, b+n) so predict and the dense sweep see identical inputs
        b, n = 5_000_017, 3001
        X = ospace.values_of(ospace.decode(np.arange(b, b + n, dtype=np.uint64), workloads.radices("cfg2")), vl)
        tp = h.predict(torch.tensor(X, dtype=torch.float32, device="cuda:0")).cpu().numpy()
        ts = h.eval_range(vl, b, b + n).cpu().numpy()
        assert np.array_equal(tp, ts), f"{prec}: {np.count_nonzero(tp != ts)} rows differ"
        e = rel_err(tp, osweep.times(model, vl, b, b + n), model["y_scale"])
        assert e.max() <= TOL[prec], f"{prec}: max rel err {e.max():.3e}"
        assert h.predict(torch.zeros((0, 14), dtype=torch.float32, device="cuda:0")).numel() == 0


# ------------------------------------------------------------------ top-k
def test_tiny_top1_exact_fp32(pk):
    vl = workloads.space("tiny")
    model = workloads.load_model("tiny_14-32-32-1")
    h = _handle(pk, model, "fp32")
    idx, t, cnt = h.sweep(vl, 1)
    ri, rt = osweep.topk(model, vl, 1)
    assert cnt == 1 and int(idx[0]) == int(ri[0])
    assert rel_err(t.cpu().numpy(), rt, model["y_scale"]).max() <= TOL["fp32"]


@pytest.mark.parametrize("prec,k", [("fp32", 16), ("bf16", 16), ("tf32", 64), ("bf16", 1024), ("fp32", 1000),
                                    ("fp16", 16), ("fp16", 1024), ("fp32_3xtf32", 64)])
def test_cfg2_subrange_topk(pk, prec, k):
    vl = workloads.space("cfg2")
    model = workloads.load_model("cfg2_14-128-128-1")
    h = _handle(pk, model, prec)
    b, e = 33_333_333, 33_333_333 + (1 << 21) + 55
    idx, t, cnt = h.sweep(vl, k, b, e)
    ri, rt = osweep.topk(model, vl, k, b, e)
    assert cnt == k
    check_topk(idx.cpu().numpy().astype(np.uint64), t.cpu().numpy(), ri, rt,
               lambda i: osweep.times_at(model, vl, i), TOL[prec], model["y_scale"])


@pytest.mark.parametrize("prec", ["bf16", "fp16", "fp32", "fp32_3xtf32"])
def test_cfg2_full_sweep_reevaluated(pk, prec):
    vl = workloads.space("cfg2")
    model = workloads.load_model("cfg2_14-128-128-1")
    h = _handle(pk, model, prec)
    idx, t, cnt = h.sweep(vl, 16)
    idx = idx.cpu().numpy().astype(np.uint64)
    t = t.cpu().numpy()
    assert cnt == 16 and np.all(np.diff(t) >= 0)
    e = rel_err(t, osweep.times_at(model, vl, idx), model["y_scale"])
    assert e.max() <= TOL[prec]


def test_all_ties_net_full_size(pk):
    vl = workloads.space("cfg5")
    model = workloads.all_ties_net(vl, [128, 128])
    h = _handle(pk, model, "bf16")
    b = 9_000_000_000
    idx, t, _ = h.sweep(vl, 64, b, b + 3_000_000)
    assert idx.cpu().numpy().tolist() == list(range(b, b + 64))


@pytest.mark.parametrize("prec", ["fp32", "bf16", "fp16"])
def test_affine_net_closed_form_full_cfg5(pk, prec):
    vl = workloads.space("cfg5")
    model = workloads.affine_net(vl, [128, 128], seed=11)
    h = _handle(pk, model, prec)
    k = 256
    idx, t, _ = h.sweep(vl, k)
    ci, ct = pins.affine_kbest(model, vl, k)
    C, tables = pins.affine_tables(model, vl)
    digits = ospace.decode(idx.cpu().numpy().astype(np.uint64), workloads.radices("cfg5"))

    def closed(ii):
        d = ospace.decode(np.asarray(ii, np.uint64), workloads.radices("cfg5"))
        return C + sum(tables[j][d[:, j]] for j in range(14))

    assert digits.shape == (k, 14)
    check_topk(idx.cpu().numpy().astype(np.uint64), t.cpu().numpy(), np.array(ci, np.uint64), np.array(ct),
               closed, TOL[prec], model["y_scale"])


def test_edge_cases(pk):
    vl = workloads.space("cfg2")
    model = workloads.load_model("cfg2_14-128-128-1")
    h = _handle(pk, model, "bf16")
    # empty range
    idx, t, cnt = h.sweep(vl, 8, 1000, 1000)
    assert cnt == 0
    # k larger than the range, ragged single partial tile
    idx, t, cnt = h.sweep(vl, 50, 1000, 1007)
    assert cnt == 7 and sorted(idx[:7].cpu().tolist()) == list(range(1000, 1007))
    assert np.all(idx[7:].cpu().numpy() == -1)
    # invalid arguments raise
    with pytest.raises(pk.SurrogateError):
        h.sweep(vl, 0)
    with pytest.raises(pk.SurrogateError):
        h.sweep(vl, 2000)
    with pytest.raises(pk.SurrogateError):
        h.sweep(vl, 4, 10, 5)


def test_shard_invariance_bitwise(pk):
    vl = workloads.space("cfg2")
    model = workloads.load_model("cfg2_14-128-128-1")
    h = _handle(pk, model, "bf16")
    b, e, k = 1_000_000, 1_000_000 + 4_000_003, 32
    full_i, full_t, _ = h.sweep(vl, k, b, e)
    for W in (2, 3, 8):
        recs = []
        for r in range(W):
            lo, hi = ospace.shard(e - b, W, r)
            recs.append(h.sweep_records(vl, k, b + lo, b + hi))
        mi, mt, _ = h.merge_topk(torch.cat(recs), W, k, k)
        assert torch.equal(mi, full_i) and torch.equal(mt, full_t)


# ------------------------------------------------------------------ ensemble (cfg4)
@pytest.mark.parametrize("device", ["C2075", "V100"])
def test_cfg4_ensemble_combined_model(pk, device):
    vl = workloads.space("cfg2")
    model = workloads.with_device(workloads.load_model("cfg4_17-128-128-1_x8"),
                                  workloads.device_features("onehot", device))
    assert len(model["members"]) == 8 and model["widths"][0] == 17
    h = _handle(pk, model, "bf16")
    b, n = 77_777_777, (1 << 18) + 13
    t = h.eval_range(vl, b, b + n).cpu().numpy()
    ref = osweep.times(model, vl, b, b + n)
    assert rel_err(t, ref, model["y_scale"]).max() <= TOL["bf16"]
    idx, tk, cnt = h.sweep(vl, 16, b, b + n)
    ri, rt = osweep.topk(model, vl, 16, b, b + n)
    check_topk(idx.cpu().numpy().astype(np.uint64), tk.cpu().numpy(), ri, rt,
               lambda i: osweep.times_at(model, vl, i), TOL["bf16"], model["y_scale"])
    # explicit batch through the same ensemble passes
    X = ospace.values_of(ospace.decode(np.arange(b, b + 2000, dtype=np.uint64), workloads.radices("cfg2")), vl)
    tp = h.predict(torch.tensor(X, dtype=torch.float32, device="cuda:0")).cpu().numpy()
    assert np.array_equal(tp, t[:2000])


def test_ensemble_fp32_path_and_chunking(pk):
    # 3 random members on the FP32 path: 1e-5 against the oracle's mean
    vl = workloads.space("cfg5")
    model = workloads.random_net(vl, [64, 64], seed=21, ensemble=3)
    h = _handle(pk, model, "fp32")
    b, n = 5_000_000_000, 300_001
    t = h.eval_range(vl, b, b + n).cpu().numpy()
    ref = osweep.times(model, vl, b, b + n)
    assert rel_err(t, ref, model["y_scale"]).max() <= TOL["fp32"]


# ------------------------------------------------------------------ CTA pairs (cfg3, H = 256)
@pytest.mark.parametrize("prec", ["bf16", "fp16"])
@pytest.mark.parametrize("hidden", [[256], [256, 256], [256, 256, 256]])
def test_pair_kernel_random_nets(pk, hidden, prec):
    # cta_group::2 kernel over ragged ranges (odd pair-tile counts, tails inside rank 1)
    vl = workloads.space("cfg3")
    model = workloads.random_net(vl, hidden, seed=len(hidden) + 40)
    h = _handle(pk, model, prec)
    for b, n in [(0, 256 * 148 * 2 + 129), (1_279_000_000 - 70_001, 70_001), (5, 3)]:
        t = h.eval_range(vl, b, b + n).cpu().numpy()
        ref = osweep.times(model, vl, b, b + n)
        e = rel_err(t, ref, model["y_scale"])
        assert e.max() <= TOL[prec], f"{hidden} [{b},{b + n}): max rel err {e.max():.3e}"


@pytest.mark.parametrize("prec", ["bf16", "fp16"])
def test_cfg3_trained_slice_and_topk(pk, prec):
    vl = workloads.space("cfg3")
    model = workloads.load_model("cfg3_14-256-256-256-1")
    h = _handle(pk, model, prec)
    b, n = 640_000_017, (1 << 18) + 333
    t = h.eval_range(vl, b, b + n).cpu().numpy()
    ref = osweep.times(model, vl, b, b + n)
    assert rel_err(t, ref, model["y_scale"]).max() <= TOL[prec]
    idx, tk, cnt = h.sweep(vl, 64, b, b + n)
    ri, rt = osweep.topk(model, vl, 64, b, b + n)
    assert cnt == 64
    check_topk(idx.cpu().numpy().astype(np.uint64), tk.cpu().numpy(), ri, rt,
               lambda i: osweep.times_at(model, vl, i), TOL[prec], model["y_scale"])
    X = ospace.values_of(ospace.decode(np.arange(b, b + 3000, dtype=np.uint64), workloads.radices("cfg3")), vl)
    tp = h.predict(torch.tensor(X, dtype=torch.float32, device="cuda:0")).cpu().numpy()
    assert np.array_equal(tp, t[:3000])


@pytest.mark.parametrize("prec", ["bf16", "fp16"])
def test_cfg3_full_sweep_reevaluated(pk, prec):
    vl = workloads.space("cfg3")
    model = workloads.load_model("cfg3_14-256-256-256-1")
    h = _handle(pk, model, prec)
    idx, t, cnt = h.sweep(vl, 64)
    idx = idx.cpu().numpy().astype(np.uint64)
    t = t.cpu().numpy()
    assert cnt == 64 and np.all(np.diff(t) >= 0)
    assert rel_err(t, osweep.times_at(model, vl, idx), model["y_scale"]).max() <= TOL[prec]


# ------------------------------------------------------------------ the paper's space
@pytest.mark.parametrize("b,n", [(358318080000000 - 300_001, 300_001), (123_456_789_012_345, (1 << 18) + 3)])
def test_paper_space_window_times(pk, b, n):
    # 10/12-value lists: quadruple decoder table of 117 KB, indices near 3.58e14
    vl = workloads.space("paper")
    model = workloads.load_model("paper_14-128-128-1")
    h = _handle(pk, model, "bf16")
    t = h.eval_range(vl, b, b + n).cpu().numpy()
    ref = osweep.times(model, vl, b, b + n)
    assert rel_err(t, ref, model["y_scale"]).max() <= TOL["bf16"]


def test_paper_space_window_topk1024(pk):
    vl = workloads.space("paper")
    model = workloads.load_model("paper_14-128-128-1")
    h = _handle(pk, model, "bf16")
    b, e = 200_000_000_000_000, 200_000_000_000_000 + (1 << 20) + 17
    idx, t, cnt = h.sweep(vl, 1024, b, e)
    ri, rt = osweep.topk(model, vl, 1024, b, e)
    assert cnt == 1024
    check_topk(idx.cpu().numpy().astype(np.uint64), t.cpu().numpy(), ri, rt,
               lambda i: osweep.times_at(model, vl, i), TOL["bf16"], model["y_scale"])


def test_campaign_chunked_and_resumed_equals_one_shot(pk, tmp_path):
    from paper_2306_14011_b200 import campaign as cp
    vl = workloads.space("cfg2")
    model = workloads.load_model("cfg2_14-128-128-1")
    h = _handle(pk, model, "bf16")
    N = 170_859_375
    full_i, full_t, _ = h.sweep(vl, 16)
    path = str(tmp_path / "c.npz")
    a = cp.for_surrogate(h, vl, 16, 0, N, 20_000_000, path, every=2, tag="cfg2/bf16")
    a.run(max_chunks=5)
    assert not a.finished
    b = cp.for_surrogate(h, vl, 16, 0, N, 20_000_000, path, every=2, tag="cfg2/bf16")
    assert b.resumed_from == 80_000_000
    idx, t = cp.records_to_result(b.run().cpu().numpy(), 16)
    assert np.array_equal(idx, full_i.cpu().numpy().astype(np.uint64))
    assert np.array_equal(t, full_t.cpu().numpy())


@pytest.mark.parametrize("prec", ["bf16", "fp16"])
def test_predict_staged_rows_large_batch(pk, prec):
    # full tiles through the bulk-copy row staging, a ragged tail read directly,
    # and a 16-byte-misaligned x (direct reads throughout): all bitwise equal
    # (14-128-128-1: the predict instantiation of sweep_kernel8)
    vl = workloads.space("cfg2")
    model = workloads.load_model("cfg2_14-128-128-1")
    h = _handle(pk, model, prec)
    b, n = 33_000_001, (1 << 20) + 77
    X = ospace.values_of(ospace.decode(np.arange(b, b + n + 1, dtype=np.uint64), workloads.radices("cfg2")), vl)
    xb = torch.tensor(X, dtype=torch.float32, device="cuda:0")
    tp = h.predict(xb[:n]).cpu().numpy()
    ts = h.eval_range(vl, b, b + n).cpu().numpy()
    assert np.array_equal(tp, ts)
    tm = h.predict(xb[1:]).cpu().numpy()          # rows start 56 B into the buffer
    assert np.array_equal(tm, np.concatenate([ts[1:], h.eval_range(vl, b + n, b + n + 1).cpu().numpy()]))
    sample = np.random.default_rng(3).integers(0, n, 4000)
    ref = osweep.times_at(model, vl, (b + sample).astype(np.uint64))
    assert rel_err(tp[sample], ref, model["y_scale"]).max() <= TOL[prec]


# ------------------------------------------------------------------ precisions (FP16, 3xFP16 FP32 path)
@pytest.mark.parametrize("prec", ["fp16", "fp32", "bf16"])
def test_cfg5_trained_slices_and_topk1024(pk, prec):
    # the cfg5 net (the headline space of the 8-GPU sweep) on ragged windows at
    # both ends of the u64 index range, plus a k = 1024 sub-range top-k
    vl = workloads.space("cfg5")
    model = workloads.load_model("cfg5_14-128-128-1")
    h = _handle(pk, model, prec)
    for b, n in [(0, (1 << 18) + 5), (13_492_928_512 - 200_003, 200_003), (6_746_464_256, 1 << 18)]:
        t = h.eval_range(vl, b, b + n).cpu().numpy()
        e = rel_err(t, osweep.times(model, vl, b, b + n), model["y_scale"])
        assert e.max() <= TOL[prec], f"{prec} [{b}, {b + n}): max rel err {e.max():.3e}"
    b, e_ = 9_876_543_210, 9_876_543_210 + (1 << 20) + 99
    idx, tk, cnt = h.sweep(vl, 1024, b, e_)
    ri, rt = osweep.topk(model, vl, 1024, b, e_)
    assert cnt == 1024
    check_topk(idx.cpu().numpy().astype(np.uint64), tk.cpu().numpy(), ri, rt,
               lambda i: osweep.times_at(model, vl, i), TOL[prec], model["y_scale"])


def test_fp32_path_kernel_choice(pk):
    # H <= 128: 3xFP16 on kind::f16 at any depth (deeper nets: ping-pong regions
    # in the 2-slot kernel); 3xTF32 only when forced
    vl = workloads.space("cfg2")
    h = _handle(pk, workloads.load_model("cfg2_14-128-128-1"), "fp32")
    assert h.arith()[:2] == ("f16", 3)
    assert _handle(pk, workloads.load_model("cfg2_14-128-128-1"), "fp32_3xtf32").arith()[:2] == ("tf32", 3)
    assert _handle(pk, workloads.load_model("cfg2_14-128-128-1"), "fp16").arith()[:2] == ("f16", 1)
    for hidden in ([64, 64, 64], [128, 128, 128], [32, 32, 32, 32]):
        deep = workloads.random_net(vl, hidden, seed=5 + len(hidden))
        h = _handle(pk, deep, "fp32")
        assert h.arith()[:2] == ("f16", 3)
        b, n = 100_000_003, 70_001
        t = h.eval_range(vl, b, b + n).cpu().numpy()
        assert rel_err(t, osweep.times(deep, vl, b, b + n), deep["y_scale"]).max() <= TOL["fp32"], hidden
        idx, tk, cnt = h.sweep(vl, 16, b, b + n)
        ri, rt = osweep.topk(deep, vl, 16, b, b + n)
        check_topk(idx.cpu().numpy().astype(np.uint64), tk.cpu().numpy(), ri, rt,
                   lambda i: osweep.times_at(deep, vl, i), TOL["fp32"], deep["y_scale"])
    h = _handle(pk, workloads.random_net(vl, [64, 64, 64], seed=8), "fp32_3xtf32")
    assert h.arith()[:2] == ("tf32", 3)
    # issued tensor work of the cfg2 net: 16-bit L1 + (H + 16) x H bias-folded L2
    assert _handle(pk, workloads.load_model("cfg2_14-128-128-1"), "fp16").arith()[2] == 2 * (16 * 128 + 144 * 128)


@pytest.mark.parametrize("prec", ["fp16", "fp32"])
def test_fp16_range_guard(pk, prec):
    # activations that can exceed 65504 over the space are refused (SURR_E_RANGE),
    # the same net runs on BF16 / 3xTF32
    vl = workloads.space("cfg2")
    model = workloads.random_net(vl, [128, 128], seed=9)
    big = dict(model)
    big["members"] = [dict(m) for m in model["members"]]
    m0 = big["members"][0]
    m0["W"] = [w.copy() for w in m0["W"]]
    m0["W"][0] = m0["W"][0] * 1e5   # |W1| <= 2e4 loads; the bound on h1 exceeds 65504
    h = _handle(pk, big, prec)
    with pytest.raises(pk.SurrogateError, match="FP16"):
        h.sweep(vl, 4, 0, 1000)
    safe = "bf16" if prec == "fp16" else "fp32_3xtf32"
    t = _handle(pk, big, safe).eval_range(vl, 0, 1000).cpu().numpy()
    assert rel_err(t, osweep.times(big, vl, 0, 1000), big["y_scale"]).max() <= TOL[safe] * 10


@pytest.mark.parametrize("prec", ["fp32", "fp32_3xtf32", "tf32", "fp16", "bf16"])
@pytest.mark.parametrize("hidden", [[32], [64], [128], [32, 32], [64, 64]])
def test_shallow_and_narrow_nets(pk, prec, hidden):
    # one hidden layer (14-H-1: the final layer reads the layer-1 accumulator) and
    # narrow two-layer nets (N-halves of 16 / 32 columns) on ragged ranges
    vl = workloads.space("cfg2")
    model = workloads.random_net(vl, hidden, seed=sum(hidden) + len(hidden))
    h = _handle(pk, model, prec)
    for b, n in [(0, 148 * 2 * 128 + 77), (170859375 - 40_001, 40_001)]:
        t = h.eval_range(vl, b, b + n).cpu().numpy()
        e = rel_err(t, osweep.times(model, vl, b, b + n), model["y_scale"])
        assert e.max() <= TOL[prec], f"{prec} {hidden} [{b}, {b + n}): max rel err {e.max():.3e}"
    idx, tk, cnt = h.sweep(vl, 32, 1_000_003, 1_000_003 + 300_000)
    ri, rt = osweep.topk(model, vl, 32, 1_000_003, 1_000_003 + 300_000)
    check_topk(idx.cpu().numpy().astype(np.uint64), tk.cpu().numpy(), ri, rt,
               lambda i: osweep.times_at(model, vl, i), TOL[prec], model["y_scale"])


# ------------------------------------------------------------------ full BASELINE sizes, bench launch configuration
def _full_sweep_checks(pk, model, vl, prec, k, sample_seed):
    """Full-space sweep as bench.py runs it: every returned item re-evaluated by
    the oracle (within tol, sorted), and a property that holds at any size: no
    sampled config the top-k left out is faster than the k-th time by more than
    the tie band."""
    h = _handle(pk, model, prec)
    idx, t, cnt = h.sweep(vl, k)
    idx = idx.cpu().numpy().astype(np.uint64)
    t = t.cpu().numpy()
    assert cnt == k and np.all(np.diff(t) >= 0) and len(set(idx.tolist())) == k
    assert rel_err(t, osweep.times_at(model, vl, idx), model["y_scale"]).max() <= TOL[prec]
    N = int(np.prod([len(v) for v in vl]))
    rng = np.random.default_rng(sample_seed)
    sample = np.unique(rng.integers(0, N, 1 << 17, dtype=np.uint64))
    ts = osweep.times_at(model, vl, sample)
    Tk = float(t[-1])
    band = 2 * TOL[prec] * abs(Tk)
    missing = sample[(ts < Tk - band) & ~np.isin(sample, idx)]
    assert missing.size == 0, f"{missing.size} sampled configs faster than the k-th time are not in the top-k"


@pytest.mark.parametrize("prec", ["fp16", "fp32"])
def test_cfg5_full_sweep_reevaluated_and_sampled(pk, prec):
    vl = workloads.space("cfg5")
    _full_sweep_checks(pk, workloads.load_model("cfg5_14-128-128-1"), vl, prec, 1024, 5)


def test_cfg4_full_sweep_reevaluated_and_sampled(pk):
    vl = workloads.space("cfg2")
    model = workloads.with_device(workloads.load_model("cfg4_17-128-128-1_x8"),
                                  workloads.device_features("onehot", "V100"))
    _full_sweep_checks(pk, model, vl, "fp16", 16, 4)


def test_cfg2_full_sweep_sampled_property(pk):
    vl = workloads.space("cfg2")
    _full_sweep_checks(pk, workloads.load_model("cfg2_14-128-128-1"), vl, "fp16", 16, 2)


# ------------------------------------------------------------------ scalers, device-feature encodings, NaN order
@pytest.mark.parametrize("prec", ["fp16", "fp32"])
def test_minmax_and_standard_scalers(pk, prec):
    # the kernel implements the generic affine map z = (x - shift) / scale,
    # so StandardScaler and min-max run through the same path
    from oracle import scaler
    vl = workloads.space("cfg2")
    X = workloads.predict_rows(vl, 5000, seed=3)
    for fit in (scaler.fit_standard, scaler.fit_minmax):
        model = workloads.random_net(vl, [128, 128], seed=17)
        model["x_shift"], model["x_scale"] = fit(X)
        h = _handle(pk, model, prec)
        b, n = 12_345_678, 150_001
        t = h.eval_range(vl, b, b + n).cpu().numpy()
        e = rel_err(t, osweep.times(model, vl, b, b + n), model["y_scale"])
        assert e.max() <= TOL[prec], f"{fit.__name__} {prec}: {e.max():.3e}"


def test_cfg4_gflops_encoding(pk):
    # the device feature as DP GFLOPS instead of one-hot; a
    # random 15-input ensemble whose constant feature is folded into b_1
    vl = workloads.space("cfg2")
    base = workloads.random_net(vl + [[513.0, 4700.0, 7500.0]], [128, 128], seed=19, ensemble=2)
    model = workloads.with_device(base, workloads.device_features("gflops", "P100"))
    assert model["widths"][0] == 15
    h = _handle(pk, model, "fp16")
    b, n = 50_000_001, 100_003
    t = h.eval_range(vl, b, b + n).cpu().numpy()
    assert rel_err(t, osweep.times(model, vl, b, b + n), model["y_scale"]).max() <= TOL["fp16"]


def test_nan_predictions_rank_last_by_index(pk):
    # NaN times order after +inf, ties by index: an all-NaN net's
    # top-k is the first k indices of the range, times NaN.  Non-finite weights
    # are refused at load, so the NaN comes from the arithmetic: a target scale
    # of 1e40 (finite in float64) overflows the FP32 output weights to inf, and
    # inf x relu(0) = NaN in every row of the all-ties net
    vl = workloads.space("cfg2")
    model = workloads.all_ties_net(vl, [128, 128])
    model["members"][0]["W"][-1][:] = 0.5
    model["y_scale"] = 1e40
    for prec in ("fp16", "fp32"):
        h = _handle(pk, model, prec)
        idx, t, cnt = h.sweep(vl, 8, 777, 777 + 5000)
        assert idx.cpu().tolist() == list(range(777, 785))
        assert torch.isnan(t).all()


# ------------------------------------------------------------------ cfg2 full enumeration
def _golden(name, k):
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", f"{name}_full_top{k}_oracle.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (scripts/make_golden_topk.py)")
    return json.load(open(path))


@pytest.mark.parametrize("prec,k", [("fp32", 16), ("fp32", 64), ("fp16", 16), ("fp16", 64), ("bf16", 16),
                                    ("fp32_3xtf32", 16)])
def test_cfg2_full_space_topk_vs_oracle_enumeration(pk, prec, k):
    # the whole 15^7 space on the GPU against the oracle's float64 enumeration of
    # every config (tests/golden/cfg2_full_top64_oracle.json, written by
    # scripts/make_golden_topk.py from oracle/ only): G17 acceptance
    g = _golden("cfg2", 64)
    vl = workloads.space("cfg2")
    model = workloads.load_model(g["weights"])
    h = _handle(pk, model, prec)
    idx, t, cnt = h.sweep(vl, k)
    assert cnt == k
    ri = np.array(g["idx"][:k], np.uint64)
    rt = np.array(g["t"][:k])
    check_topk(idx.cpu().numpy().astype(np.uint64), t.cpu().numpy(), ri, rt,
               lambda i: osweep.times_at(model, vl, i), TOL[prec], model["y_scale"])
    if prec.startswith("fp32"):
        # the FP32 path's "exact top-k": the same set as the oracle unless oracle
        # times tie within the tolerance at the k-th place
        Tk = float(rt[-1])
        gpu = set(idx.cpu().numpy().astype(np.uint64).tolist())
        for i, ti in zip(ri.tolist(), rt.tolist()):
            assert i in gpu or abs(ti - Tk) <= 2 * TOL[prec] * Tk


def test_cfg4_full_space_topk_vs_oracle_enumeration(pk):
    # the 8-member combined-GPU ensemble (17 inputs, one-hot V100) over the whole
    # cfg2 space against the oracle's float64 enumeration (golden file)
    g = _golden("cfg4", 16)
    vl = workloads.space("cfg2")
    model = workloads.with_device(workloads.load_model(g["weights"]),
                                  workloads.device_features(g["device"][0], g["device"][1]))
    for prec in ("fp16", "fp32"):
        h = _handle(pk, model, prec)
        idx, t, cnt = h.sweep(vl, 16)
        check_topk(idx.cpu().numpy().astype(np.uint64), t.cpu().numpy(), np.array(g["idx"], np.uint64),
                   np.array(g["t"]), lambda i: osweep.times_at(model, vl, i), TOL[prec], model["y_scale"])


def test_non_default_stream_ordering(pk):
    # the calls are stream-ordered on the caller's stream: the same results on a
    # side stream (work queued behind a long kernel on that stream) as on the default one
    vl = workloads.space("cfg2")
    model = workloads.load_model("cfg2_14-128-128-1")
    h = _handle(pk, model, "fp16")
    ref_i, ref_t, _ = h.sweep(vl, 16, 5_000_000, 9_000_000)
    dense_ref = h.eval_range(vl, 1_000, 201_000)
    X = torch.tensor(workloads.predict_rows(vl, 50_000, seed=4), dtype=torch.float32, device="cuda:0")
    pred_ref = h.predict(X)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        busy = torch.randn(4096, 4096, device="cuda:0")
        for _ in range(8):
            busy = busy @ busy / 64.0  # keeps the side stream busy while the calls are queued
        i2, t2, _ = h.sweep(vl, 16, 5_000_000, 9_000_000, stream=side)
        d2 = h.eval_range(vl, 1_000, 201_000, stream=side)
        p2 = h.predict(X, stream=side)
    side.synchronize()
    assert torch.equal(i2, ref_i) and torch.equal(t2, ref_t)
    assert torch.equal(d2, dense_ref) and torch.equal(p2, pred_ref)


def test_space_change_while_sweeps_are_queued(pk):
    # a sweep queued on a busy stream keeps its value table when the next call
    # (same handle) switches to another space; the new weights of a reload do not
    # leak into sweeps queued before it either
    vl_a = workloads.space("cfg2")
    vl_b = [list(np.asarray(v) * 2.0) for v in vl_a]  # same radices, other values
    model = workloads.load_model("cfg2_14-128-128-1")
    h = _handle(pk, model, "fp16")
    ref_a = h.eval_range(vl_a, 0, 1 << 20).clone()
    ref_b = h.eval_range(vl_b, 0, 1 << 20).clone()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        busy = torch.randn(4096, 4096, device="cuda:0")
        for _ in range(8):
            busy = busy @ busy / 64.0
        ta = h.eval_range(vl_a, 0, 1 << 20, stream=side)
        tb = h.eval_range(vl_b, 0, 1 << 20, stream=side)
    side.synchronize()
    assert torch.equal(ta, ref_a) and torch.equal(tb, ref_b)
