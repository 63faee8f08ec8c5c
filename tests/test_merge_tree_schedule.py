"""Host-side model of the fused grid merge's CTA tree (a9; sweep_kernel.cuh
grid_merge_tail): CTA c's list sits in slot c; at level l node j covers CTAs
[j 2^l, (j + 1) 2^l) and lives in slot j 2^l; of two siblings the second to
arrive (per-node ticket) merges both into the left slot and climbs, a node
without a sibling climbs unmerged, the CTA that completes the root writes the
result.  The model runs the same index arithmetic under random completion
orders and checks that every CTA's list reaches the root exactly once, that a
slot is only overwritten after both of its inputs were read, and that every
ticket is re-armed (back to zero) when the launch ends."""

import random

import pytest

TREE_NODES_PER_LEVEL = 256


def run_tree(grid: int, order: list[int]):
    slots = {c: frozenset([c]) for c in range(grid)}  # slot -> set of CTA lists merged into it
    tickets = {}
    # each CTA is a coroutine-like state (node, nodes, level); a CTA blocked on a
    # ticket as first arriver simply exits, so the schedule is the arrival order
    # of CTAs at their tickets: simulate CTAs one step (one level) at a time in a
    # random interleaving driven by `order`
    state = {c: (c, grid, 0) for c in range(grid)}
    active = list(order)
    result = None
    rng = random.Random(grid * 7919 + len(order))
    while active:
        c = active[rng.randrange(len(active))] if len(active) > 1 else active[0]
        node, nodes, l = state[c]
        if nodes == 1:  # root done by this CTA
            assert result is None
            result = slots[0]
            active.remove(c)
            continue
        if (node ^ 1) < nodes:
            key = l * TREE_NODES_PER_LEVEL + (node >> 1)
            assert key < 9 * TREE_NODES_PER_LEVEL
            t = tickets.get(key, 0)
            tickets[key] = t + 1
            if t + 1 == 1:  # first arriver: exits, the sibling merges
                active.remove(c)
                continue
            tickets[key] = 0  # re-armed by the second arriver
            left, right = (node & ~1) << l, (node | 1) << l
            merged = slots[left] | slots[right]
            assert not (slots[left] & slots[right]), "a list merged twice"
            slots[left] = merged
        state[c] = (node >> 1, (nodes + 1) >> 1, l + 1)
    assert result is not None
    return result, tickets


@pytest.mark.parametrize("grid", [1, 2, 3, 4, 5, 7, 8, 37, 74, 147, 148, 255, 256])
def test_every_list_reaches_the_root_once(grid):
    rng = random.Random(grid)
    for _ in range(20):
        order = list(range(grid))
        rng.shuffle(order)
        result, tickets = run_tree(grid, order)
        assert result == frozenset(range(grid))
        assert all(v == 0 for v in tickets.values()), "a ticket was left armed"


def test_levels_fit_the_ticket_array():
    # the host allocates 9 levels x 256 tickets; grids above 256 CTAs use K2 instead
    for grid in range(1, 257):
        levels, nodes = 0, grid
        while nodes > 1:
            levels += 1
            nodes = (nodes + 1) >> 1
        assert levels <= 9
