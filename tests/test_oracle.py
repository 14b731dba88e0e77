"""Pins for the CPU oracle (-m "not gpu").  Every expected value comes from the
paper's definitions restated independently in tests/pins.py, from the cited
golden fixtures, or from mathematics (closed forms, brute force, metamorphic
relations) -- never from the oracle itself or from the CUDA path.
"""
import json
import os

import numpy as np
import pytest

import oracle
from synth import volumes as V
from tests import pins

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def solve(c, delta, algo="dinic", **kw):
    r = oracle.colgraph_solve(np.asarray(c, np.int32), delta, algo=algo, **kw)
    assert r["checks"] == oracle.ALL_CHECKS, f"invariant bits {r['checks']:#x}"
    return r


# ---------------------------------------------------------------- generic max-flow core

@pytest.mark.parametrize("ex", GOLDEN["graph_examples"], ids=lambda e: e["name"])
@pytest.mark.parametrize("algo", ["dinic", "ek", "pr"])
def test_graph_examples(ex, algo):
    r = oracle.graph_maxflow(ex["nn"], ex["arcs"], ex["s"], ex["t"], algo)
    assert r["status"] == 0 and r["flow"] == ex["flow"] and r["checks"] == oracle.ALL_CHECKS


@pytest.mark.parametrize("algo", ["dinic", "ek", "pr"])
def test_graph_random_vs_bruteforce_mincut(algo):
    """Theorem 1: max flow = min cut over all 2^(n-2) cuts; the
    residual-reachable set equals the intersection of all minimum source sets."""
    rng = np.random.default_rng(7)
    for trial in range(150):
        nn = int(rng.integers(2, 9))
        m = int(rng.integers(0, 3 * nn))
        arcs = []
        for _ in range(m):
            u, v = rng.integers(0, nn, 2)
            if u != v:
                arcs.append((int(u), int(v), int(rng.integers(0, 6))))
        s, t = 0, nn - 1
        best, minimal = pins.brute_force_mincut(nn, arcs, s, t)
        r = oracle.graph_maxflow(nn, arcs, s, t, algo)
        assert r["flow"] == best, (trial, arcs)
        assert np.array_equal(r["source_side"], minimal), (trial, arcs)
        assert r["checks"] == oracle.ALL_CHECKS


# ---------------------------------------------------------------- column-graph worked examples

@pytest.mark.parametrize("ex", GOLDEN["column_examples"], ids=lambda e: e["name"])
@pytest.mark.parametrize("algo", ["dinic", "ek", "pr"])
def test_column_examples(ex, algo):
    c = np.array(ex["c"], np.int32)
    r = solve(c, ex["delta"], algo)
    assert r["status"] == 0
    assert r["flow"] == ex["flow"]
    assert np.array_equal(r["surface"], np.array(ex["surface"], np.int32))
    if "K0" in ex:
        assert pins.k0(c) == ex["K0"]
        assert pins.surface_cost(c, r["surface"]) == ex["min_cost"]
    if "source_set_size" in ex:
        assert int(r["mask"].sum()) == ex["source_set_size"]
    if "w" in ex:  # weight mode with the printed weights reproduces the cost-mode answer
        rw = solve(np.array(ex["w"], np.int32), ex["delta"], algo, input_is_weight=True)
        assert rw["flow"] == ex["flow"] and np.array_equal(rw["surface"], r["surface"])


def test_surface_enumerator_counts():
    sc = GOLDEN["surface_counts"]
    for d, cnt in sc["by_delta"].items():
        assert len(pins.enumerate_surfaces(sc["X"], sc["Y"], sc["Z"], int(d))) == cnt


# ---------------------------------------------------------------- brute force over every feasible surface

def _check_vs_bruteforce(c, delta, algo="dinic"):
    best, lowest, _, _ = pins.brute_force_surfaces(c, delta)
    r = solve(c, delta, algo)
    assert r["status"] == 0
    assert r["flow"] == best + pins.k0(c)
    assert np.array_equal(r["surface"], lowest)
    # the minimal source set is exactly the union of columns below the surface
    X, Y, Z = c.shape
    below = np.arange(Z)[None, None, :] <= lowest[:, :, None]
    assert np.array_equal(r["mask"].astype(bool), below)


@pytest.mark.parametrize("delta", [0, 1, 2])
def test_c1_cutdown_bruteforce(delta):
    """C1's 3x3x8 cut-down, every Delta-feasible surface enumerated."""
    _check_vs_bruteforce(V.c1_cutdown(), delta)


def test_random_tiny_bruteforce():
    for seed in range(1000, 1120):
        c, delta = V.tiny_case(seed)
        X, Y, Z = c.shape
        if X * Y > 9 or Z > 8:  # keep the enumeration small
            c = c[:min(X, 3), :min(Y, 3), :min(Z, 8)]
        _check_vs_bruteforce(np.ascontiguousarray(c), delta, ("dinic", "ek", "pr")[seed % 3])


def test_weight_mode_bruteforce():
    """Arbitrary signed vertex weights: min cut = min over closed sets (empty columns allowed)."""
    for seed in range(2000, 2080):
        rng = np.random.default_rng(seed)
        X, Y, Z = int(rng.integers(1, 4)), int(rng.integers(1, 3)), int(rng.integers(1, 6))
        delta = int(rng.integers(0, 3))
        w = rng.integers(-9, 10, size=(X, Y, Z)).astype(np.int32)
        val, lowest = pins.brute_force_weight_closure(w, delta)
        r = oracle.colgraph_solve(w, delta, input_is_weight=True)
        assert r["checks"] == oracle.ALL_CHECKS
        assert r["flow"] == val
        assert np.array_equal(r["surface"], lowest)
        assert r["status"] == (6 if (lowest < 0).any() else 0)


# ---------------------------------------------------------------- 1-D DP and closed forms

@pytest.mark.parametrize("shape,delta,cmax", [((40, 1, 16), 1, 255), ((1, 33, 12), 2, 9), ((64, 1, 24), 3, 3),
                                              ((25, 1, 30), 0, 255)])
def test_line_dp(shape, delta, cmax):
    c = V.tiny(77 + delta, *shape, cmax)
    opt, surf = pins.dp_line(c.reshape(-1, shape[2]), delta)
    r = solve(c, delta)
    assert r["flow"] == opt + pins.k0(c)
    assert np.array_equal(r["surface"].ravel(), surf)


@pytest.mark.parametrize("seed", range(5))
def test_closed_form_unconstrained(seed):
    c = V.tiny(300 + seed, 6, 5, 10, (3, 255)[seed % 2])
    best, surf = pins.closed_form_unconstrained(c)
    for delta in (9, 20):  # Delta >= Z-1
        r = solve(c, delta)
        assert r["flow"] == best + pins.k0(c)
        assert np.array_equal(r["surface"], surf)


@pytest.mark.parametrize("seed", range(5))
def test_closed_form_flat(seed):
    c = V.tiny(400 + seed, 5, 6, 9, (3, 255)[seed % 2])
    best, surf = pins.closed_form_flat(c)
    r = solve(c, 0)
    assert r["flow"] == best + pins.k0(c)
    assert np.array_equal(r["surface"], surf)


# ---------------------------------------------------------------- metamorphic relations

def test_metamorphic():
    c = V.generate("C1")[:8, :6, :]
    delta = 2
    base = solve(c, delta)
    assert base["flow"] == pins.surface_cost(c, base["surface"]) + pins.k0(c)
    plus = solve(c + 7, delta)
    assert plus["flow"] == base["flow"] and np.array_equal(plus["surface"], base["surface"])
    times = solve(c * 3, delta)
    assert times["flow"] == 3 * base["flow"] and np.array_equal(times["surface"], base["surface"])
    fx = solve(c[::-1].copy(), delta)
    assert fx["flow"] == base["flow"] and np.array_equal(fx["surface"], base["surface"][::-1])
    fy = solve(c[:, ::-1].copy(), delta)
    assert fy["flow"] == base["flow"] and np.array_equal(fy["surface"], base["surface"][:, ::-1])
    tr = solve(np.ascontiguousarray(c.transpose(1, 0, 2)), delta)
    assert tr["flow"] == base["flow"] and np.array_equal(tr["surface"], base["surface"].T)


def test_c1_full_value_identity():
    """On C1 itself: |f| = cost(surface) + K0, surface Delta-feasible, mask downward closed."""
    c = V.generate("C1")
    r = solve(c, 2)
    s = r["surface"]
    assert r["status"] == 0
    assert r["flow"] == pins.surface_cost(c, s) + pins.k0(c)
    assert np.abs(np.diff(s, axis=0)).max() <= 2 and np.abs(np.diff(s, axis=1)).max() <= 2
    Z = c.shape[2]
    assert np.array_equal(r["mask"].astype(bool), np.arange(Z)[None, None, :] <= s[:, :, None])
    assert r["flow"] == solve(c, 2, "ek")["flow"]


def test_invalid_inputs():
    assert oracle.colgraph_solve(np.zeros((1, 1, 1), np.int32), -1)["status"] == 1
    assert oracle.graph_maxflow(2, [(0, 1, 1)], 0, 0)["status"] == 1


# ---------------------------------------------------------------- NEXT-3: anisotropic smoothness (Delta_x != Delta_y)
# The edge interval is defined per adjacent column; SURVEY.md §8(f) NEXT-3.

def test_aniso_random_tiny_bruteforce():
    """Every (Delta_x, Delta_y)-feasible surface enumerated: |f| = min cost + K0 and the
    surface is the pointwise-lowest optimum."""
    rng = np.random.default_rng(31)
    for trial in range(120):
        X, Y, Z = int(rng.integers(1, 4)), int(rng.integers(1, 4)), int(rng.integers(1, 8))
        dx, dy = (int(v) for v in rng.integers(0, 4, 2))
        c = rng.integers(0, (4, 10, 256)[trial % 3], size=(X, Y, Z)).astype(np.int32)
        _check_vs_bruteforce(c, (dx, dy), "dinic" if trial % 2 else "ek")


def test_aniso_weight_mode_bruteforce():
    rng = np.random.default_rng(32)
    for trial in range(60):
        X, Y, Z = int(rng.integers(1, 4)), int(rng.integers(1, 3)), int(rng.integers(1, 6))
        dx, dy = (int(v) for v in rng.integers(0, 3, 2))
        w = rng.integers(-9, 10, size=(X, Y, Z)).astype(np.int32)
        val, lowest = pins.brute_force_weight_closure(w, (dx, dy))
        r = oracle.colgraph_solve(w, (dx, dy), input_is_weight=True)
        assert r["checks"] == oracle.ALL_CHECKS
        assert r["flow"] == val and np.array_equal(r["surface"], lowest)


@pytest.mark.parametrize("dx,dy", [(1, 0), (2, 5), (0, 3)])
def test_aniso_lines(dx, dy):
    """Y = 1: only Delta_x constrains the line; X = 1: only Delta_y (Viterbi DP)."""
    c = V.tiny(90 + dx, 30, 1, 14, 255)
    opt, surf = pins.dp_line(c.reshape(-1, 14), dx)
    r = solve(c, (dx, dy))
    assert r["flow"] == opt + pins.k0(c) and np.array_equal(r["surface"].ravel(), surf)
    c = V.tiny(95 + dy, 1, 27, 12, 9)
    opt, surf = pins.dp_line(c.reshape(-1, 12), dy)
    r = solve(c, (dx, dy))
    assert r["flow"] == opt + pins.k0(c) and np.array_equal(r["surface"].ravel(), surf)


@pytest.mark.parametrize("seed", range(4))
def test_aniso_closed_form_rows(seed):
    """Delta_x >= Z-1, Delta_y = 0: every x-slice is one flat row, independently of the
    others -- S(x, .) = lowest argmin_z sum_y c(x,y,z)."""
    c = V.tiny(500 + seed, 5, 4, 9, (3, 255)[seed % 2])
    tot = c.astype(np.int64).sum(axis=1)  # [x][z]
    z = tot.argmin(axis=1)
    r = solve(c, (8, 0))
    assert r["flow"] == int(tot.min(axis=1).sum()) + pins.k0(c)
    assert np.array_equal(r["surface"], np.repeat(z[:, None], 4, axis=1).astype(np.int32))


def test_aniso_transpose_swaps_deltas():
    c = V.generate("C1")[:7, :5, :]
    a = solve(c, (1, 3))
    b = solve(np.ascontiguousarray(c.transpose(1, 0, 2)), (3, 1))
    assert a["flow"] == b["flow"] and np.array_equal(a["surface"], b["surface"].T)
    assert solve(c, (2, 2))["flow"] == solve(c, 2)["flow"]


# ---------------------------------------------------------------- NEXT-1: soft smoothness (convex penalty)
# VCE-weight net surface: cost sum c(x,y,S) + sum over 4-neighbour pairs of
# f(|S(p) - S(q)|), f convex with f(0) = 0, |dS| <= Delta still hard.

def _random_convex(rng, K):
    inc = np.sort(rng.integers(0, 12, K))  # non-decreasing increments -> convex f
    return np.cumsum(inc).astype(np.int32)


def test_soft_random_tiny_bruteforce():
    rng = np.random.default_rng(51)
    for trial in range(150):
        X, Y, Z = int(rng.integers(1, 4)), int(rng.integers(1, 4)), int(rng.integers(1, 8))
        dx, dy = (int(v) for v in rng.integers(0, 4, 2))
        pen = _random_convex(rng, max(dx, dy, 1))
        c = rng.integers(0, (4, 10, 256)[trial % 3], size=(X, Y, Z)).astype(np.int32)
        best, lowest = pins.brute_force_soft(c, (dx, dy), pen)
        r = oracle.colgraph_solve(c, (dx, dy), algo="dinic" if trial % 2 else "ek", penalty=pen)
        assert r["checks"] == oracle.ALL_CHECKS, trial
        assert r["flow"] == best + pins.k0(c), (trial, r["flow"], best + pins.k0(c))
        assert np.array_equal(r["surface"], lowest), trial


@pytest.mark.parametrize("delta", [1, 3, 6])
def test_soft_line_dp(delta):
    rng = np.random.default_rng(52 + delta)
    pen = _random_convex(rng, delta)
    c = V.tiny(600 + delta, 40, 1, 14, 255)
    opt, surf = pins.dp_line_soft(c.reshape(-1, 14), delta, pen)
    r = solve(c, delta, penalty=pen)
    assert r["flow"] == opt + pins.k0(c) and np.array_equal(r["surface"].ravel(), surf)


def test_soft_zero_penalty_is_hard():
    c = V.generate("C1")[:6, :5, :]
    a, b = solve(c, 2), solve(c, 2, penalty=[0, 0])
    assert a["flow"] == b["flow"] and np.array_equal(a["mask"], b["mask"])


def test_soft_linear_penalty_limit():
    """A penalty steeper than any cost difference forces a flat-in-pairs optimum: with
    f(d) = M*d and M > 255*Z the optimal surface is flat (every |dS| >= 1 costs more than any
    column can save)."""
    c = V.tiny(77, 4, 3, 9, 255)
    M = 255 * 9 + 1
    r = solve(c, 3, penalty=[M, 2 * M, 3 * M])
    tot = c.astype(np.int64).sum(axis=(0, 1))
    assert (r["surface"] == int(tot.argmin())).all()
    assert r["flow"] == int(tot.min()) + pins.k0(c)


def test_soft_rejects_nonconvex():
    c = np.zeros((2, 2, 4), np.int32)
    assert oracle.colgraph_solve(c, 2, penalty=[5, 6])["status"] == 1   # f(2)-2f(1)+f(0) < 0
    assert oracle.colgraph_solve(c, 3, penalty=[1, 2])["status"] == 1   # too short


@pytest.mark.parametrize("seed", range(40))
def test_push_relabel_algorithm_pins(seed):
    """The oracle's third max-flow algorithm (two-phase FIFO push-relabel, §2.1) on random
    tiny volumes (brute force), weight mode (brute-force closures) and general intervals + bands."""
    rng = np.random.default_rng(9000 + seed)
    c, delta = V.tiny_case(9000 + seed)
    c = np.ascontiguousarray(c[:3, :3, :8])
    _check_vs_bruteforce(c, delta, "pr")
    X, Y, Z = (int(v) for v in rng.integers(1, 4, 3))
    w = rng.integers(-9, 10, size=(X, Y, Z)).astype(np.int32)
    dd = int(rng.integers(0, 3))
    best, lowest = pins.brute_force_weight_closure(w, dd)
    r = oracle.colgraph_solve(w, dd, input_is_weight=True, algo="pr")
    assert r["checks"] == oracle.ALL_CHECKS and r["flow"] == best
    d4 = tuple(int(v) for v in rng.integers(0, 4, 4))
    best, low, _ = pins.brute_force_general(c, d4)
    r = oracle.colgraph_solve(c, d4, algo="pr")
    assert r["checks"] == oracle.ALL_CHECKS and r["flow"] == best + pins.k0(c) and np.array_equal(r["surface"], low)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_push_relabel_agrees_with_dinic(name):
    from synth import volumes as V2
    spec = V2.CONFIGS[name]
    c = V2.generate(name)
    a = oracle.colgraph_solve(c, spec.delta, algo="pr")
    b = oracle.colgraph_solve(c, spec.delta, algo="dinic")
    assert a["checks"] == b["checks"] == oracle.ALL_CHECKS
    assert a["flow"] == b["flow"] and np.array_equal(a["mask"], b["mask"])
