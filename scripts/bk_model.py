"""Sequential Python model of k_bk_stage (csrc/bk.cuh), lane loops written out, for debugging the
algorithm on a CPU box: python scripts/bk_model.py [ncases] compares it with the oracle (so does
tests/test_bk_model.py).  Not product code: the library never calls it."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from synth import volumes as V  # noqa: E402

FREE, S, T = 0, 1, 2
INQ = 4
TERM, ORPHAN, NOPAR = 10, 11, 15
INF = 2**31 - 1


def zo_of(z, d):
    return 0 if z == 0 else (z - d if z > d else -1)


def zi_of(z, d, Z):
    return 0 if z == 0 else (z + d if z + d < Z else -1)


class Model:
    def __init__(self, c, delta):
        X, Y, Z = c.shape
        self.X, self.Y, self.Z = X, Y, Z
        self.dl = [delta] * 4
        n = X * Y * Z
        w = np.zeros((X, Y, Z), np.int64)
        w[:, :, 0] = c[:, :, 0] - (c.sum(axis=2) + 1)
        w[:, :, 1:] = c[:, :, 1:] - c[:, :, :-1]
        w = w.ravel()
        self.E = np.maximum(-w, 0).astype(np.int64)
        self.T = np.maximum(w, 0).astype(np.int64)
        self.T0 = self.T.sum()
        self.D = np.zeros(n, np.int64)
        self.L = np.zeros((4, n), np.int64)
        self.H = np.zeros(n, np.int64)
        self.ts = np.zeros(n, np.int64)
        self.dist = np.ones(n, np.int64)
        self.next = -np.ones(n, np.int64)
        self.onext = -np.ones(n, np.int64)
        for v in range(n):
            e, t = self.E[v], self.T[v]
            self.H[v] = (S | (TERM << 4)) if e > 0 else (T | (TERM << 4)) if t > 0 else (FREE | (NOPAR << 4))
        self.time = [1, 1]

    def xyz(self, v):
        col, z = divmod(v, self.Z)
        x, y = divmod(col, self.Y)
        return x, y, z

    def nbr(self, seg, v, k):
        x, y, z = self.xyz(v)
        if k == 0:
            return v - 1 if z >= 1 else -1
        if k == 1:
            return v + 1 if z + 1 < self.Z else -1
        d = (k - 2) & 3
        nx = x + (d == 0) - (d == 1)
        ny = y + (d == 2) - (d == 3)
        x0, x1, y0, y1 = seg
        if nx < x0 or nx >= x1 or ny < y0 or ny >= y1:
            return -1
        zz = zo_of(z, self.dl[d]) if k < 6 else zi_of(z, self.dl[d ^ 1], self.Z)
        if zz < 0:
            return -1
        return (nx * self.Y + ny) * self.Z + zz

    def step(self, v, k):
        return self.nbr((0, self.X, 0, self.Y), v, k)

    def res_fwd(self, v, k, u):
        if k == 1:
            return self.D[u]
        if k >= 6:
            return self.L[(k - 6) ^ 1][u]
        return INF

    def res_rev(self, v, k, u):
        if k == 0:
            return self.D[v]
        if 2 <= k < 6:
            return self.L[k - 2][v]
        return INF

    def push(self, v, k, u, f, fwd):
        if k == 0:
            self.D[v] += f if fwd else -f
        elif k == 1:
            self.D[u] += -f if fwd else f
        elif k < 6:
            self.L[k - 2][v] += f if fwd else -f
        else:
            self.L[(k - 6) ^ 1][u] += -f if fwd else f


def rev_code(k):
    return 1 if k == 0 else 0 if k == 1 else (6 + ((k - 2) ^ 1) if k < 6 else 2 + ((k - 6) ^ 1))


def tree(h):
    return h & 3


def par(h):
    return (h >> 4) & 15


def with_par(h, p):
    return (h & ~(15 << 4)) | (p << 4)


def stage(m, seg, axis, half):
    aq, oq = [], []  # python lists in place of the linked lists
    TIME = m.time[0]
    x0, x1, y0, y1 = seg
    cx0, cx1, cy0, cy1 = x0, x1, y0, y1
    if axis == 0:
        if x0 + half >= x1:
            cx1 = cx0
        else:
            cx0, cx1 = x0 + half - 1, x0 + half + 1
    elif axis == 1:
        if y0 + half >= y1:
            cy1 = cy0
        else:
            cy0, cy1 = y0 + half - 1, y0 + half + 1
    for x in range(cx0, cx1):
        for y in range(cy0, cy1):
            for z in range(m.Z):
                v = (x * m.Y + y) * m.Z + z
                h = m.H[v]
                if tree(h) != FREE and not (h & INQ):
                    m.H[v] = h | INQ
                    aq.append(v)
    cur = -1
    while True:
        if cur >= 0 and tree(m.H[cur]) == FREE:
            cur = -1
        while cur < 0 and aq:
            v = aq.pop(0)
            m.H[v] &= ~INQ
            if tree(m.H[v]) != FREE:
                cur = v
        if cur < 0:
            break
        X = tree(m.H[cur])
        lanes = []
        for k in range(10):
            u = m.nbr(seg, cur, k)
            cap = 0
            hu = 0
            if u >= 0:
                cap = m.res_fwd(cur, k, u) if X == S else m.res_rev(cur, k, u)
                if cap > 0:
                    hu = m.H[u]
            lanes.append((k, u, cap, hu))
        seen = set()
        for k, u, cap, hu in lanes:
            if u >= 0 and cap > 0 and tree(hu) == FREE and u not in seen:
                seen.add(u)
                m.H[u] = X | INQ | (rev_code(k) << 4)
                m.ts[u] = m.ts[cur]
                m.dist[u] = m.dist[cur] + 1
                if not (hu & INQ):
                    aq.append(u)
        meet = [(k, u) for k, u, cap, hu in lanes if u >= 0 and cap > 0 and tree(hu) not in (FREE, X)]
        if not meet:
            cur = -1
            continue
        k, u = meet[0]
        augment(m, oq, cur, k, u, X)
        TIME += 1
        while oq:
            p = oq.pop(0)
            hp = m.H[p]
            Xp = tree(hp)
            cands = []
            info = []
            for kk in range(10):
                w = m.nbr(seg, p, kk)
                hw, capa = 0, 0
                if w >= 0:
                    hw = m.H[w]
                    if tree(hw) == Xp:
                        capa = m.res_rev(p, kk, w) if Xp == S else m.res_fwd(p, kk, w)
                dd = None
                if capa > 0 and par(hw) != ORPHAN:
                    j, steps = w, 0
                    while True:
                        if m.ts[j] == TIME:
                            dd = steps + m.dist[j]
                            break
                        pj = par(m.H[j])
                        steps += 1
                        if pj == TERM:
                            dd = steps
                            break
                        if pj >= ORPHAN:
                            break
                        assert steps < 10**6
                        j = m.step(j, pj)
                info.append((kk, w, hw, capa))
                if dd is not None:
                    cands.append((dd, kk, w))
            if cands:
                dd, kk, w = min(cands)
                m.H[p] = with_par(hp, kk)
                m.ts[p] = TIME
                m.dist[p] = dd + 1
                m.ts[w] = TIME
                m.dist[w] = dd
                continue
            grp = {}
            for kk, w, hw, capa in info:
                if w >= 0 and tree(hw) == Xp:
                    act = capa > 0 and not (hw & INQ)
                    orp = par(hw) == rev_code(kk)
                    a0, o0, h0 = grp.get(w, (False, False, hw))
                    grp[w] = (a0 or act, o0 or orp, h0)
            for w, (act, orp, hw) in grp.items():
                h = hw
                if act:
                    h |= INQ
                if orp:
                    h = with_par(h, ORPHAN)
                m.H[w] = h
                if act:
                    aq.append(w)
                if orp:
                    oq.append(w)
            m.H[p] = FREE | (hp & INQ) | (NOPAR << 4)
    m.time[1] = max(m.time[1], TIME)


def augment(m, oq, i, k, u, X):
    if X == S:
        sa, tb, f = i, u, m.res_fwd(i, k, u)
    else:
        sa, tb, f = u, i, m.res_rev(i, k, u)
    j = sa
    while True:
        pc = par(m.H[j])
        if pc == TERM:
            f = min(f, m.E[j])
            break
        assert pc < ORPHAN
        q = m.step(j, pc)
        f = min(f, m.res_rev(j, pc, q))
        j = q
    j = tb
    while True:
        pc = par(m.H[j])
        if pc == TERM:
            f = min(f, m.T[j])
            break
        assert pc < ORPHAN
        q = m.step(j, pc)
        f = min(f, m.res_fwd(j, pc, q))
        j = q
    assert f > 0
    m.push(i, k, u, f, X == S)

    def orphan(j):
        m.H[j] = with_par(m.H[j], ORPHAN)
        oq.append(j)
    j = sa
    while True:
        pc = par(m.H[j])
        if pc == TERM:
            m.E[j] -= f
            if m.E[j] == 0:
                orphan(j)
            break
        q = m.step(j, pc)
        m.push(j, pc, q, f, False)
        if m.res_rev(j, pc, q) == 0:
            orphan(j)
        j = q
    j = tb
    while True:
        pc = par(m.H[j])
        if pc == TERM:
            m.T[j] -= f
            if m.T[j] == 0:
                orphan(j)
            break
        q = m.step(j, pc)
        m.push(j, pc, q, f, True)
        if m.res_fwd(j, pc, q) == 0:
            orphan(j)
        j = q


def solve(c, delta, bx, by):
    m = Model(c, delta)
    X, Y = m.X, m.Y
    sx, sy, axis, half, prefer_x = min(bx, X), min(by, Y), -1, 0, True
    while True:
        nsx, nsy = -(-X // sx), -(-Y // sy)
        for b in range(nsx * nsy):
            x0 = (b % nsx) * sx
            y0 = (b // nsx) * sy
            stage(m, (x0, min(X, x0 + sx), y0, min(Y, y0 + sy)), axis, half)
        m.time[0] = m.time[1] + 1
        if nsx == 1 and nsy == 1:
            break
        if nsx > 1 and (prefer_x or nsy <= 1):
            half, sx, axis = sx, sx * 2, 0
        else:
            half, sy, axis = sy, sy * 2, 1
        prefer_x = not prefer_x
    assert (m.E >= 0).all() and (m.T >= 0).all() and (m.D >= 0).all() and (m.L >= 0).all()
    return int(m.T0 - m.T.sum())


if __name__ == "__main__":
    import oracle  # the check below only (test infrastructure)
    rng = np.random.default_rng(1)
    ncase = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    for seed in range(3000, 3000 + ncase):
        c, delta = V.tiny_case(seed)
        bx, by = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        f = solve(c, delta, bx, by)
        o = oracle.colgraph_solve(c, delta)
        assert f == o["flow"], (seed, f, o["flow"], c.shape, delta, bx, by)
    print("ok", ncase)
