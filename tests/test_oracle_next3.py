"""Oracle pins for the rest of NEXT-3: general proper-ordered edge intervals
(PAPER.md:42 -- the edge interval of a vertex toward each adjacent column; here possibly asymmetric,
S(q) - S(p) in [-d(+x), d(-x)] for q = p + x) and narrow bands (PAPER.md:456, 475 -- the surface of a
column confined to [lo, hi), reading R15).  Each result is checked against brute-force enumeration of
every feasible surface (tests/pins.py), never against the oracle itself."""
import numpy as np
import pytest

import oracle
from tests import pins


def rand_band(rng, X, Y, Z, delta, tries=200):
    """A random band (X, Y, 2) satisfying the consistency precondition for `delta`."""
    for _ in range(tries):
        lo = rng.integers(0, Z, size=(X, Y))
        hi = lo + rng.integers(1, Z + 1, size=(X, Y))
        hi = np.minimum(hi, Z)
        band = np.stack([lo, hi], axis=-1).astype(np.int32)
        if pins.band_consistent(band, delta):
            return band
    return None


@pytest.mark.parametrize("seed", range(80))
def test_asymmetric_intervals_bruteforce(seed):
    rng = np.random.default_rng(7000 + seed)
    X, Y, Z = int(rng.integers(1, 4)), int(rng.integers(1, 4)), int(rng.integers(1, 7))
    c = rng.integers(0, int(rng.choice([3, 9, 255])) + 1, size=(X, Y, Z)).astype(np.int32)
    d4 = tuple(int(v) for v in rng.integers(0, 4, size=4))
    best, lowest, nfeas = pins.brute_force_general(c, d4)
    assert nfeas > 0
    r = oracle.colgraph_solve(c, d4)
    assert r["status"] == 0 and r["checks"] == oracle.ALL_CHECKS
    assert r["flow"] == best + pins.k0(c), (d4, r["flow"], best)
    assert np.array_equal(r["surface"], lowest), d4
    assert np.array_equal(r["mask"], (np.arange(Z)[None, None, :] <= lowest[..., None]).astype(np.uint8))


@pytest.mark.parametrize("seed", range(20))
def test_asymmetric_mirror(seed):
    """Flipping x exchanges the +x and -x intervals (and y likewise): same value, mirrored surface."""
    rng = np.random.default_rng(7200 + seed)
    X, Y, Z = int(rng.integers(2, 5)), int(rng.integers(2, 5)), int(rng.integers(2, 9))
    c = rng.integers(0, 50, size=(X, Y, Z)).astype(np.int32)
    a, b, e, f = (int(v) for v in rng.integers(0, 4, size=4))
    r = oracle.colgraph_solve(c, (a, b, e, f))
    rx = oracle.colgraph_solve(c[::-1].copy(), (b, a, e, f))
    ry = oracle.colgraph_solve(c[:, ::-1].copy(), (a, b, f, e))
    assert r["flow"] == rx["flow"] == ry["flow"]
    assert np.array_equal(r["surface"][::-1], rx["surface"])
    assert np.array_equal(r["surface"][:, ::-1], ry["surface"])


def test_symmetric_four_tuple_is_the_isotropic_case():
    rng = np.random.default_rng(7300)
    for _ in range(20):
        c = rng.integers(0, 30, size=(3, 4, 7)).astype(np.int32)
        d, dy = int(rng.integers(0, 4)), int(rng.integers(0, 4))
        a = oracle.colgraph_solve(c, (d, d, dy, dy))
        b = oracle.colgraph_solve(c, (d, dy))
        assert a["flow"] == b["flow"] and np.array_equal(a["mask"], b["mask"])


def test_one_sided_interval_is_monotone():
    """d(+x) = 0 and d(-x) = Z: S may only rise along +x (S(x+1) >= S(x)); on a line the lowest
    optimum is then non-decreasing -- and a cost volume whose column minima fall along x forces
    the compromise the brute force finds."""
    rng = np.random.default_rng(7400)
    for _ in range(10):
        X, Z = 5, 6
        c = rng.integers(0, 40, size=(X, 1, Z)).astype(np.int32)
        r = oracle.colgraph_solve(c, (0, Z, 0, 0))
        s = r["surface"][:, 0]
        assert (np.diff(s) >= 0).all()
        best, lowest, _ = pins.brute_force_general(c, (0, Z, 0, 0))
        assert r["flow"] == best + pins.k0(c) and np.array_equal(r["surface"], lowest)


@pytest.mark.parametrize("seed", range(80))
def test_band_bruteforce(seed):
    rng = np.random.default_rng(7500 + seed)
    X, Y, Z = int(rng.integers(1, 4)), int(rng.integers(1, 4)), int(rng.integers(2, 8))
    c = rng.integers(0, int(rng.choice([3, 9, 255])) + 1, size=(X, Y, Z)).astype(np.int32)
    d4 = tuple(int(v) for v in rng.integers(0, 4, size=4)) if seed % 2 else int(rng.integers(0, 4))
    band = rand_band(rng, X, Y, Z, d4)
    if band is None:
        pytest.skip("no consistent band drawn")
    best, lowest, nfeas = pins.brute_force_general(c, d4, band)
    assert nfeas > 0
    r = oracle.colgraph_solve(c, d4, band=band)
    assert r["status"] == 0 and r["checks"] == oracle.ALL_CHECKS
    assert r["flow"] == best + pins.k0_band(c, band), (band.tolist(), r["flow"], best)
    assert np.array_equal(r["surface"], lowest)
    assert ((r["surface"] >= band[..., 0]) & (r["surface"] < band[..., 1])).all()
    # the basement below the band is in S, the attic above the surface is not
    assert np.array_equal(r["mask"], (np.arange(Z)[None, None, :] <= lowest[..., None]).astype(np.uint8))


def test_full_band_is_the_plain_graph():
    rng = np.random.default_rng(7700)
    for _ in range(20):
        X, Y, Z = 3, 3, 8
        c = rng.integers(0, 60, size=(X, Y, Z)).astype(np.int32)
        band = np.zeros((X, Y, 2), np.int32)
        band[..., 1] = Z
        a = oracle.colgraph_solve(c, 2, band=band)
        b = oracle.colgraph_solve(c, 2)
        assert a["flow"] == b["flow"] and np.array_equal(a["mask"], b["mask"])


def test_band_of_height_one_fixes_the_surface():
    rng = np.random.default_rng(7800)
    X, Y, Z = 3, 4, 9
    c = rng.integers(0, 60, size=(X, Y, Z)).astype(np.int32)
    lo = np.full((X, Y), 4, np.int32)
    band = np.stack([lo, lo + 1], axis=-1)
    r = oracle.colgraph_solve(c, 1, band=band)
    assert (r["surface"] == 4).all()
    assert r["flow"] == int(c[:, :, 4].sum()) + pins.k0_band(c, band)


def test_band_rejections():
    c = np.zeros((2, 2, 5), np.int32)
    bad = np.zeros((2, 2, 2), np.int32)  # lo == hi
    assert oracle.colgraph_solve(c, 1, band=bad)["status"] == 1
    band = np.zeros((2, 2, 2), np.int32)
    band[..., 1] = 6  # hi > Z
    assert oracle.colgraph_solve(c, 1, band=band)["status"] == 1
    band[..., 1] = 5
    assert oracle.colgraph_solve(c, 1, input_is_weight=True, band=band)["status"] == 1
