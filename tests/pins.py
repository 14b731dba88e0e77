"""Independent pins for the oracle (test code; no shared arithmetic with oracle/ or the CUDA path).

Each function restates, from the mathematics, a result the oracle must
reproduce:
  * brute_force_surfaces -- every Delta-feasible net surface of a tiny volume
    (§1.2: a net surface "intersects with each column at exactly
    one vertex"; adjacent tops differ by at most Delta), its cost
    sum_cols c(x,y,S(x,y)), the minimum and the pointwise-lowest optimum.
  * k0 -- the construction constant of SURVEY.md §8(c) "Closed form for the
    value": |f| = min_S cost(S) + K0,
    K0 = sum_cols [ sum_{z>=1} max(0, c(z-1) - c(z)) - c(0) ], derived from
    the cut capacity (Eq. 6) of the closed set {z <= S(x,y)} under
    the weights w(0) = c(0) - (sum c + 1), w(z) = c(z) - c(z-1).
  * dp_line -- exact Viterbi DP for Y = 1 (or X = 1) volumes.
  * closed-form cases Delta >= Z-1 (independent columns) and Delta = 0 (flat).
  * soft smoothness (NEXT-1, PAPER.md:42-43 VCE-weight net surface): brute force and line DP
    with the cost sum c(x,y,S) + sum over 4-neighbour pairs of f(|S(p) - S(q)|).
  * general edge intervals and narrow bands (NEXT-3; PAPER.md:42 proper ordering, PAPER.md:456
    narrow bands): surfaces with S(q) - S(p) in [-d(+x), d(-x)] for q = p + x (likewise y) and
    S(p) in [lo(p), hi(p)); k0_band restates the construction constant for the band rule.
  * brute_force_mincut -- all s-t cuts of a small general graph (PAPER.md
    Eq. 6 and Theorem 1), their minimum and the intersection of all minimum
    source sets (the minimal source set).
"""
from __future__ import annotations

import itertools

import numpy as np


def _pair_ok(a, b, delta, allow_empty):
    ok = (np.abs(a.astype(np.int64) - b.astype(np.int64)) <= delta) & (a >= 0) & (b >= 0)
    if allow_empty:
        ok |= (a < 0) & (b < 0)
    return ok


def _dxy(delta):
    """delta: int (isotropic) or (delta_x, delta_y) -- the edge interval toward x- and
    y-neighbours."""
    return (int(delta[0]), int(delta[1])) if isinstance(delta, (tuple, list)) else (int(delta), int(delta))


def _d4(delta):
    """(+x, -x, +y, -y) edge intervals: int, (dx, dy) or a 4-tuple."""
    if isinstance(delta, (tuple, list)) and len(delta) == 4:
        return tuple(int(d) for d in delta)
    dx, dy = _dxy(delta)
    return (dx, dx, dy, dy)


def enumerate_surfaces_general(X: int, Y: int, Z: int, delta, band=None) -> np.ndarray:
    """All feasible top assignments (K, X*Y) under the general interval: for q = p + x,
    S(p) - S(q) <= d(+x) (p's arc toward +x) and S(q) - S(p) <= d(-x) (q's arc toward -x); the same
    with y.  band (X, Y, 2): S(p) in [lo, hi)."""
    dpx, dmx, dpy, dmy = _d4(delta)
    cur = np.zeros((1, 0), dtype=np.int16)
    for col in range(X * Y):
        x, y = divmod(col, Y)
        lo, hi = (int(band[x, y, 0]), int(band[x, y, 1])) if band is not None else (0, Z)
        vals = np.arange(lo, hi, dtype=np.int16)
        K = cur.shape[0]
        new = np.repeat(cur, len(vals), axis=0)
        v = np.tile(vals, K).astype(np.int64)
        ok = np.ones(len(v), dtype=bool)
        if x > 0:
            p = new[:, (x - 1) * Y + y].astype(np.int64)
            ok &= (p - v <= dpx) & (v - p <= dmx)
        if y > 0:
            p = new[:, x * Y + y - 1].astype(np.int64)
            ok &= (p - v <= dpy) & (v - p <= dmy)
        cur = np.concatenate([new[ok], v[ok, None].astype(np.int16)], axis=1)
    return cur


def brute_force_general(c: np.ndarray, delta, band=None):
    """(min cost, lowest optimal surface, number of feasible surfaces) under general intervals / bands."""
    X, Y, Z = c.shape
    S = enumerate_surfaces_general(X, Y, Z, delta, band)
    cols = c.reshape(X * Y, Z).astype(np.int64)
    cost = cols[np.arange(X * Y)[None, :], S.astype(np.int64)].sum(axis=1)
    best = cost.min()
    opt = S[cost == best]
    return int(best), opt.min(axis=0).reshape(X, Y).astype(np.int32), int(len(S))


def k0_band(c: np.ndarray, band) -> int:
    """|f| = min cost + K0 under the band rule: the cut of the closed set {z <= S(p)} is
    N + sum_{v in S} w(v) (Eq. 6 with source capacities -w, sink capacities w), the band weights
    telescope to c(p, S(p)) - (sum_{band} c + 1) per column, and N = sum max(0, -w) =
    sum_band c + 1 - c(lo) + sum_{lo<z<hi} max(0, c(z-1) - c(z)); so per column
    K0 = sum_{lo<z<hi} max(0, c(z-1) - c(z)) - c(lo)."""
    cc = c.astype(np.int64)
    lo, hi = band[..., 0].astype(np.int64), band[..., 1].astype(np.int64)
    drops = np.zeros_like(cc)
    drops[:, :, 1:] = np.maximum(0, cc[:, :, :-1] - cc[:, :, 1:])
    P = np.cumsum(drops, axis=2)  # P[z] = sum_{1 <= j <= z} drops
    take = lambda a, i: np.take_along_axis(a, i[..., None], axis=2)[..., 0]  # noqa: E731
    return int((take(P, hi - 1) - take(P, lo) - take(cc, lo)).sum())


def band_consistent(band, delta) -> bool:
    """The band reading's precondition (R15): for every neighbour pair and direction, the
    lower and the upper band limits move by no more than the edge interval allows."""
    dpx, dmx, dpy, dmy = _d4(delta)
    lo, hi = band[..., 0].astype(np.int64), band[..., 1].astype(np.int64)
    ok = True
    if band.shape[0] > 1:
        dlo, dhi = lo[1:] - lo[:-1], hi[1:] - hi[:-1]
        ok &= bool(((-dlo <= dpx) & (dlo <= dmx) & (-dhi <= dpx) & (dhi <= dmx)).all())
    if band.shape[1] > 1:
        dlo, dhi = lo[:, 1:] - lo[:, :-1], hi[:, 1:] - hi[:, :-1]
        ok &= bool(((-dlo <= dpy) & (dlo <= dmy) & (-dhi <= dpy) & (dhi <= dmy)).all())
    return ok


def enumerate_surfaces(X: int, Y: int, Z: int, delta, allow_empty: bool = False) -> np.ndarray:
    """All feasible top-assignments, shape (K, X*Y), column index x*Y + y:
    |S(x,y) - S(x-1,y)| <= delta_x and |S(x,y) - S(x,y-1)| <= delta_y.

    allow_empty adds top = -1 (empty column) for the weight-mode closure pin.
    """
    dx, dy = _dxy(delta)
    vals = np.arange(-1 if allow_empty else 0, Z, dtype=np.int16)
    cur = np.zeros((1, 0), dtype=np.int16)
    for col in range(X * Y):
        x, y = divmod(col, Y)
        K = cur.shape[0]
        new = np.repeat(cur, len(vals), axis=0)
        v = np.tile(vals, K)
        ok = np.ones(len(v), dtype=bool)
        if x > 0:
            ok &= _pair_ok(v, new[:, (x - 1) * Y + y], dx, allow_empty)
        if y > 0:
            ok &= _pair_ok(v, new[:, x * Y + y - 1], dy, allow_empty)
        cur = np.concatenate([new[ok], v[ok, None]], axis=1)
    return cur


def brute_force_surfaces(c: np.ndarray, delta):
    """(min cost, lowest optimal surface (X,Y), number of optima, number of feasible surfaces)."""
    X, Y, Z = c.shape
    S = enumerate_surfaces(X, Y, Z, delta)
    cols = c.reshape(X * Y, Z).astype(np.int64)
    cost = cols[np.arange(X * Y)[None, :], S.astype(np.int64)].sum(axis=1)
    best = cost.min()
    opt = S[cost == best]
    return int(best), opt.min(axis=0).reshape(X, Y).astype(np.int32), int(len(opt)), int(len(S))


def soft_penalty_sum(S: np.ndarray, X: int, Y: int, penalty) -> np.ndarray:
    """sum over 4-neighbour column pairs of f(|S(p) - S(q)|), f(0) = 0, f(d) = penalty[d-1];
    S: (K, X*Y) top assignments."""
    f = np.concatenate([[0], np.asarray(penalty, np.int64)])
    T = S.reshape(-1, X, Y).astype(np.int64)
    tot = np.zeros(S.shape[0], np.int64)
    if X > 1:
        tot += f[np.abs(T[:, 1:, :] - T[:, :-1, :])].sum(axis=(1, 2))
    if Y > 1:
        tot += f[np.abs(T[:, :, 1:] - T[:, :, :-1])].sum(axis=(1, 2))
    return tot


def brute_force_soft(c: np.ndarray, delta, penalty):
    """(min of sum c(S) + sum f(|dS|) over Delta-feasible surfaces, lowest optimal surface)."""
    X, Y, Z = c.shape
    S = enumerate_surfaces(X, Y, Z, delta)
    cols = c.reshape(X * Y, Z).astype(np.int64)
    cost = cols[np.arange(X * Y)[None, :], S.astype(np.int64)].sum(axis=1) + soft_penalty_sum(S, X, Y, penalty)
    best = cost.min()
    opt = S[cost == best]
    return int(best), opt.min(axis=0).reshape(X, Y).astype(np.int32)


def dp_line_soft(cl: np.ndarray, delta: int, penalty):
    """Viterbi on a line of columns with the soft penalty: (min cost, lowest optimal surface)."""
    X, Z = cl.shape
    cl = cl.astype(np.int64)
    f = np.concatenate([[0], np.asarray(penalty, np.int64)])
    big = np.iinfo(np.int64).max // 4

    def step(prev):
        out = np.full(Z, big, np.int64)
        for d in range(-delta, delta + 1):
            lo, hi = max(0, -d), min(Z, Z - d)
            if lo < hi:
                out[lo:hi] = np.minimum(out[lo:hi], prev[lo + d:hi + d] + f[abs(d)])
        return out

    F = np.zeros((X, Z), np.int64)
    B = np.zeros((X, Z), np.int64)
    F[0] = cl[0]
    for x in range(1, X):
        F[x] = cl[x] + step(F[x - 1])
    B[X - 1] = cl[X - 1]
    for x in range(X - 2, -1, -1):
        B[x] = cl[x] + step(B[x + 1])
    opt = int(F[X - 1].min())
    through = F + B - cl
    return opt, np.array([int(np.flatnonzero(through[x] == opt)[0]) for x in range(X)], np.int32)


def brute_force_weight_closure(w: np.ndarray, delta):
    """Weight mode: min over closed sets S of sum_{v in S} w(v) (plus sum max(-w,0) = min cut),
    and the pointwise-lowest optimal top assignment (-1 = empty column)."""
    X, Y, Z = w.shape
    S = enumerate_surfaces(X, Y, Z, delta, allow_empty=True)
    cols = np.concatenate([np.zeros((X * Y, 1), np.int64), np.cumsum(w.reshape(X * Y, Z).astype(np.int64), axis=1)],
                          axis=1)  # prefix sums, index top+1
    val = cols[np.arange(X * Y)[None, :], S.astype(np.int64) + 1].sum(axis=1)
    best = val.min()
    opt = S[val == best]
    const = int(np.maximum(-w.astype(np.int64), 0).sum())
    return int(best) + const, opt.min(axis=0).reshape(X, Y).astype(np.int32)


def k0(c: np.ndarray) -> int:
    c = c.astype(np.int64)
    drops = np.maximum(0, c[:, :, :-1] - c[:, :, 1:]).sum()
    return int(drops - c[:, :, 0].sum())


def surface_cost(c: np.ndarray, surf: np.ndarray) -> int:
    X, Y, Z = c.shape
    return int(np.take_along_axis(c.astype(np.int64), surf.reshape(X, Y, 1).astype(np.int64), axis=2).sum())


def dp_line(cl: np.ndarray, delta: int):
    """Exact DP on a line of columns cl[x][z]: (min cost, lowest optimal surface)."""
    X, Z = cl.shape
    cl = cl.astype(np.int64)
    big = np.iinfo(np.int64).max // 4

    def window_min(prev):
        out = np.full(Z, big, np.int64)
        for d in range(-delta, delta + 1):
            lo, hi = max(0, -d), min(Z, Z - d)
            if lo < hi:
                out[lo:hi] = np.minimum(out[lo:hi], prev[lo + d:hi + d])
        return out

    F = np.zeros((X, Z), np.int64)
    B = np.zeros((X, Z), np.int64)
    F[0] = cl[0]
    for x in range(1, X):
        F[x] = cl[x] + window_min(F[x - 1])
    B[X - 1] = cl[X - 1]
    for x in range(X - 2, -1, -1):
        B[x] = cl[x] + window_min(B[x + 1])
    opt = int(F[X - 1].min())
    through = F + B - cl
    surf = np.array([int(np.flatnonzero(through[x] == opt)[0]) for x in range(X)], np.int32)
    return opt, surf


def closed_form_unconstrained(c: np.ndarray):
    """Delta >= Z-1: columns are independent; lowest argmin per column."""
    return int(c.astype(np.int64).min(axis=2).sum()), c.argmin(axis=2).astype(np.int32)


def closed_form_flat(c: np.ndarray):
    """Delta = 0: one flat surface; lowest argmin of the per-depth total."""
    tot = c.astype(np.int64).sum(axis=(0, 1))
    z = int(tot.argmin())
    return int(tot[z]), np.full(c.shape[:2], z, np.int32)


def brute_force_mincut(nn: int, arcs, s: int, t: int):
    """(min cut value, minimal source set as bool[nn]) by enumerating all s-t cuts."""
    others = [v for v in range(nn) if v not in (s, t)]
    best, sets = None, []
    for bits in itertools.product([0, 1], repeat=len(others)):
        side = np.zeros(nn, bool)
        side[s] = True
        for v, b in zip(others, bits):
            side[v] = bool(b)
        val = sum(cap for (u, v, cap) in arcs if side[u] and not side[v])
        if best is None or val < best:
            best, sets = val, [side]
        elif val == best:
            sets.append(side)
    return best, np.logical_and.reduce(sets)
