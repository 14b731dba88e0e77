"""Negative pins of the oracle's invariant checker (oracle.c check_invariants).

Every oracle test asserts checks == ALL_CHECKS; these tests show that each bit actually clears
when the state breaks the invariant it stands for, so a checker that always returned every bit
would fail here.  The invariants: capacity 0 <= f <= c (Eq. 2), antisymmetry of the
arc pair (Eq. 3), conservation (Eq. 4), value = flow into t = flow out of s (Eq. 5),
t not in S and cut capacity == |f| with no infinite arc leaving S (Theorem 1; Eq. 6).

The state is a hand-solved 5-node network (s=0, a=1, b=2, c=3, t=4):
    s->a 10, s->b 2, a->b INF, a->t 1, b->t 4, b->c 1, c->t 1
max flow 6 (every sink arc saturated): s->a 4, s->b 2, a->b 3, a->t 1, b->t 4, b->c 1, c->t 1;
minimal source set S = {s, a, b} (s->a keeps residual 6, a->b is infinite), cut a->t + b->t + b->c = 6.
"""
import numpy as np
import pytest

import oracle

INF = 1 << 62
ARCS = [(0, 1, 10), (0, 2, 2), (1, 2, INF), (1, 4, 1), (2, 4, 4), (2, 3, 1), (3, 4, 1)]
FLOW = [4, 2, 3, 1, 4, 1, 1]
S_MARK = [1, 1, 1, 0, 0]
ALL = oracle.ALL_CHECKS
B = oracle.CHECK_BITS


def state(flow=None):
    f = list(FLOW if flow is None else flow)
    rf = [c - x for (_, _, c), x in zip(ARCS, f)]
    return rf, list(f)


def check(rf, rr, mark=S_MARK, value=6):
    return oracle.graph_check(5, ARCS, rf, rr, 0, 4, np.array(mark, np.uint8), value)


def test_hand_solved_state_passes_every_check():
    rf, rr = state()
    assert check(rf, rr) == ALL
    # and the oracle's own solve of the same network agrees with the hand solution
    r = oracle.graph_maxflow(5, ARCS, 0, 4)
    assert r["flow"] == 6 and list(r["source_side"].astype(int)) == S_MARK and r["checks"] == ALL


def test_antisymmetry_bit_clears():
    rf, rr = state()
    rr[5] += 1  # reverse slot of b->c no longer pairs with its forward residual
    got = check(rf, rr)
    assert not got & B["antisymmetry"]
    assert got == ALL & ~B["antisymmetry"]


def test_capacity_bit_clears():
    rf, rr = state()
    rf[3], rr[3] = -1, 2  # a->t carries 2 > capacity 1 (pair still consistent)
    got = check(rf, rr)
    assert not got & B["capacity"]


def test_negative_flow_clears_capacity():
    rf, rr = state()
    rf[5], rr[5] = 2, -1  # b->c carries -1
    assert not check(rf, rr) & B["capacity"]


def test_conservation_bit_clears():
    rf, rr = state([4, 2, 4, 1, 4, 1, 1])  # one more unit on a->b: a and b unbalanced
    got = check(rf, rr)
    assert got == ALL & ~B["conservation"]


def test_value_bit_clears():
    rf, rr = state()
    got = check(rf, rr, value=7)
    assert not got & B["value"]
    assert got & B["conservation"] and got & B["capacity"]


def test_t_in_source_set_clears():
    rf, rr = state()
    got = check(rf, rr, mark=[1, 1, 1, 0, 1])
    assert not got & B["t_not_in_S"]


def test_infinite_arc_across_cut_clears():
    rf, rr = state()
    got = check(rf, rr, mark=[1, 1, 0, 0, 0])  # a in S, b not: a->b (INF) leaves S
    assert got == ALL & ~B["cut_eq_flow"]


def test_cut_capacity_mismatch_clears():
    # a feasible but NOT maximum flow: cut capacity 6 != value 5 (b->c / c->t unused)
    rf, rr = state([4, 1, 3, 1, 4, 0, 0])
    got = check(rf, rr, value=5)
    assert not got & B["cut_eq_flow"]
    assert got & B["conservation"] and got & B["value"]


@pytest.mark.parametrize("seed", range(20))
def test_random_single_corruption_never_passes(seed):
    """Any single +-1 change of one residual slot of the solved state breaks some invariant."""
    rng = np.random.default_rng(seed)
    rf, rr = state()
    i = int(rng.integers(len(ARCS)))
    if rng.integers(2):
        rf[i] += int(rng.choice([-1, 1]))
    else:
        rr[i] += int(rng.choice([-1, 1]))
    assert check(rf, rr) != ALL
