"""Pins for oracle.space (cardinality, decode/encode, enumeration, sampling, split)."""

import itertools

import numpy as np
import pytest

import workloads
from oracle import space


def test_paper_cardinality(golden):
    # P:241 "10^7 x 12^7 = 3.58 x 10^14", value lists from the Table
    g = golden["gang_values"]["value"]
    v = golden["vector_values"]["value"]
    assert len(g) == 10 and len(v) == 12
    radices = [len(g), len(v)] * 7
    assert space.cardinality(radices) == golden["search_space_size"]["value"]
    assert workloads.SPACES["paper"][0] == g and workloads.SPACES["paper"][1] == v
    assert len(workloads.SPACES["paper"]) == golden["num_params"]["value"]


@pytest.mark.parametrize("name,size", [("tiny", 2 ** 14), ("cfg2", 15 ** 7), ("cfg3", 20 ** 7),
                                       ("cfg5", 28 ** 7), ("paper", 10 ** 7 * 12 ** 7)])
def test_config_cardinalities(name, size):
    assert space.cardinality(workloads.radices(name)) == size


def test_small_cardinalities():
    assert space.cardinality([10, 12]) == 120
    assert space.cardinality([10, 12, 10, 12]) == 14400
    assert space.cardinality([7]) == 7
    assert len(space.enumerate_all([[1, 2], [3]])) == 2


def test_enumeration_is_lexicographic_decode_order():
    # brute force: itertools.product enumerates in lexicographic order of value indices
    vl = [[1, 2], [3], [5, 6, 7], [8, 9]]
    radices = [len(v) for v in vl]
    allc = space.enumerate_all(vl)
    assert allc[:2] == [(1, 3, 5, 8), (1, 3, 5, 9)]
    assert len(allc) == space.cardinality(radices)
    dig = space.decode(np.arange(len(allc)), radices)
    vals = space.values_of(dig, vl)
    assert [tuple(int(x) for x in r) for r in vals] == allc


def test_decode_roundtrip_tiny_all():
    r = workloads.radices("tiny")
    idx = np.arange(2 ** 14, dtype=np.uint64)
    d = space.decode(idx, r)
    assert np.array_equal(space.encode(d, r), idx)
    # tiny space digits are the binary expansion, parameter 0 most significant
    ref = np.array(list(itertools.product([0, 1], repeat=14)))
    assert np.array_equal(d, ref)


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg5", "paper"])
def test_decode_roundtrip_random_and_python_ints(name):
    r = workloads.radices(name)
    n = space.cardinality(r)
    rng = np.random.default_rng(7)
    idx = np.unique(np.concatenate([rng.integers(0, n, 100000, dtype=np.uint64),
                                    np.array([0, 1, n - 2, n - 1], dtype=np.uint64)]))
    d = space.decode(idx, r)
    assert np.array_equal(space.encode(d, r), idx)
    # independent arbitrary-precision divmod on a subsample
    for i, row in zip(idx[::997], d[::997]):
        x = int(i)
        digs = []
        for rr in reversed(r):
            x, m = divmod(x, rr)
            digs.append(m)
        assert list(reversed(digs)) == list(row)


def test_decode_boundaries():
    r = workloads.radices("paper")
    n = space.cardinality(r)
    assert list(space.decode(0, r)) == [0] * 14
    assert list(space.decode(n - 1, r)) == [x - 1 for x in r]
    d1 = space.decode(1, r)
    assert list(d1[:-1]) == [0] * 13 and d1[-1] == 1
    with pytest.raises(ValueError):
        space.decode(n, r)


def test_sample_distinct_members_and_marginals():
    r = [10, 12, 10]
    rng = np.random.default_rng(3)
    idx = space.sample_indices(r, 1000, rng)
    assert len(set(idx.tolist())) == 1000
    assert int(idx.max()) < space.cardinality(r)
    # marginal of a 10-value parameter over 10^4 draws: +-5 pp of 10%
    idx = space.sample_indices([10, 1000, 1000], 10000, np.random.default_rng(11))
    d = space.decode(idx, [10, 1000, 1000])[:, 0]
    freq = np.bincount(d, minlength=10) / len(d)
    assert np.all(np.abs(freq - 0.1) < 0.05)
    # whole space when n == |S|
    idx = space.sample_indices([10, 12], 120, np.random.default_rng(5))
    assert sorted(idx.tolist()) == list(range(120))
    with pytest.raises(ValueError):
        space.sample_indices([2, 2], 5, np.random.default_rng(0))


def test_split_sizes(golden):
    n, ntr, nte = golden["samples_per_gpu"]["value"]
    tr, te = space.split(n, 0.75, np.random.default_rng(1))
    assert (len(tr), len(te)) == (ntr, nte)
    assert len(set(tr.tolist()) | set(te.tolist())) == n
    tr2, _ = space.split(n, 0.75, np.random.default_rng(1))
    assert np.array_equal(tr, tr2)
    tr, te = space.split(4, 0.75, np.random.default_rng(1))
    assert (len(tr), len(te)) == (3, 1)


@pytest.mark.parametrize("n,w", [(16384, 1), (16384, 3), (170859375, 8), (13492928512, 8),
                                 (7, 8), (2 ** 64 - 1, 8)])
def test_shard_partition(n, w):
    parts = [space.shard(n, w, r) for r in range(w)]
    assert parts[0][0] == 0 and parts[-1][1] == n
    for (a, b), (c, d) in zip(parts, parts[1:]):
        assert b == c
    sizes = [b - a for a, b in parts]
    assert max(sizes) - min(sizes) <= 1
