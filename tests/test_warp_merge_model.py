"""Host-side model of the per-CTA top-k list merge (a8; sweep_kernel.cuh
warp_merge): the list L (k records, sorted, its first nv valid, the rest
sentinels) and a warp's cnt <= 64 candidates are merged into the other buffer
O.  Each candidate goes to rank(c) + ub(c), ub(c) = #{valid L < c}; each valid
L[i] goes to i + #{j : ub_j <= i} (a pointer walk over the ascending ub);
O's tail beyond nv + cnt must already be sentinels (the second buffer is
sentinel-filled at the first merge).  The model runs the same arithmetic,
lane by lane, over random merge sequences and checks the list against a
plain sort of everything offered so far."""

import random

import pytest

SENT = (0xFFFFFFFF, (1 << 64) - 1)


def model_merge(L, nv, cand, k, O):
    cnt = len(cand)
    ranks = [sum(1 for o in cand if o < c) for c in cand]
    ub = [sum(1 for x in L[:nv] if x < c) for c in cand]  # upper bound over the valid prefix
    if nv == 0:
        for i in range(cnt, k):
            O[i] = SENT
    for c, r, u in zip(cand, ranks, ub):
        if r + u < k:
            O[r + u] = c
    ub_sorted = [0] * cnt
    for r, u in zip(ranks, ub):
        ub_sorted[r] = u
    for lane in range(32):
        jp = 0
        for i in range(lane, nv, 32):
            while jp < cnt and ub_sorted[jp] <= i:
                jp += 1
            if i + jp < k:
                O[i + jp] = L[i]
    return min(nv + cnt, k)


@pytest.mark.parametrize("k", [1, 2, 16, 33, 64, 100, 1024])
def test_merges_keep_the_exact_top_k(k):
    rng = random.Random(k)
    bufs = [[SENT] * k, [None] * k]  # buffer 1 starts uninitialised (garbage), as on the device
    cur, nv = 0, 0
    seen = []
    used = set()
    for _ in range(60):
        cnt = rng.randint(1, 64)
        cand = []
        while len(cand) < cnt:
            key, idx = rng.randrange(1 << 12), rng.randrange(1 << 40)  # key ties, distinct (key, idx)
            if (key, idx) not in used:
                used.add((key, idx))
                cand.append((key, idx))
        seen += cand
        O = bufs[cur ^ 1]
        nv = model_merge(bufs[cur], nv, cand, k, O)
        cur ^= 1
        expect = sorted(seen)[:k]
        assert bufs[cur][:len(expect)] == expect
        assert all(x == SENT for x in bufs[cur][len(expect):])
        assert nv == len(expect)
