"""Design study for the global relabel (a2/a5): how many rounds does a column-scan fixpoint need?

Runs on a GPU box.  For a config, solve with max_sweeps = s for a few s (mid-solve residual
states), export the state, and compute the exact reverse-BFS distances to t in plain torch with
three schemes, all exact (Bellman-Ford from INF):
  * column Jacobi: each round every column recomputes its exact in-column distances (prefix-min
    up the infinite down arcs, segmented suffix-min down the residual up arcs) from its neighbours'
    labels of the previous round; rounds until nothing changes; "worklist" = columns with a
    neighbour that changed in the previous round.
  * tile Gauss-Seidel: tiles of TX x TY columns iterate column Jacobi locally (neighbours inside
    the tile current, outside frozen for the round) until locally converged; global rounds until
    nothing changes.
It also reports the BFS depth (max finite label = levels of the level-synchronous BFS).
The final solved state's labels are checked against the library's own BFS labels (exported H).

    python scripts/relabel_study.py C4 64,256,512
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_17026_b200 import colgraph as cg  # noqa: E402
from synth import volumes as V  # noqa: E402

BIG = 1 << 40


def shift(a, d, fill):
    """value of a at the neighbour column in direction d (0:+x 1:-x 2:+y 3:-y); fill outside."""
    out = torch.full_like(a, fill)
    if d == 0:
        out[:-1] = a[1:]
    elif d == 1:
        out[1:] = a[:-1]
    elif d == 2:
        out[:, :-1] = a[:, 1:]
    else:
        out[:, 1:] = a[:, :-1]
    return out


def at_zo(a, delta, fill):
    """out[z] = a[zo(z)]: zo(0) = 0, zo(z) = z - delta (z > delta), else none"""
    out = torch.full_like(a, fill)
    Z = a.shape[-1]
    out[..., 0] = a[..., 0]
    if delta + 1 < Z:
        out[..., delta + 1:] = a[..., 1:Z - delta]
    return out


def at_zi(a, delta, fill):
    """out[z] = a[zi(z)]: zi(0) = 0, zi(z) = z + delta (z + delta < Z), else none"""
    out = torch.full_like(a, fill)
    Z = a.shape[-1]
    out[..., 0] = a[..., 0]
    if 1 + delta < Z:
        out[..., 1:Z - delta] = a[..., 1 + delta:]
    return out


class Problem:
    def __init__(self, st, X, Y, Z, delta, INF):
        E, H, T, D, L0, L1, L2, L3 = [p.view(X, Y, Z) for p in st.view(8, -1)]
        self.H = H
        self.INF = INF
        self.Z = Z
        self.delta = delta
        self.seed = torch.where(T > 0, 1, INF).to(torch.int64)
        zz = torch.arange(Z, device=st.device, dtype=torch.int64)
        self.zz = zz
        # up-chain segment ids: brk(z) = 1 if z cannot step up to z+1 (D(z+1) == 0 or top)
        brk = torch.ones_like(T, dtype=torch.int64)
        brk[..., :-1] = (D[..., 1:] <= 0).to(torch.int64)
        self.sid = torch.flip(torch.cumsum(torch.flip(brk, [-1]), -1), [-1])
        L = [L0, L1, L2, L3]
        # lateral-in reverse arc v -> u = (nbr_d, zi(z)) has residual L_{d^1}(u)
        self.inres = [at_zi(shift(L[d ^ 1], d, 0), delta, 0) > 0 for d in range(4)]
        self.has_nbr = [shift(torch.ones_like(T, dtype=torch.bool), d, False) for d in range(4)]

    def ext(self, d_cur, d_frozen=None, same_tile=None):
        """min over t-arc and lateral out-arcs of 1 + label(target)"""
        e = self.seed.clone()
        INF = self.INF
        for d in range(4):
            nb = shift(d_cur, d, INF)
            if d_frozen is not None:
                nb = torch.where(same_tile[d], nb, shift(d_frozen, d, INF))
            lo = at_zo(nb, self.delta, INF)
            li = torch.where(self.inres[d], at_zi(nb, self.delta, INF), INF)
            e = torch.minimum(e, torch.minimum(lo, li) + 1)
        return e

    def colsolve(self, ext):
        """exact in-column distances given ext: prefix-min up the down arcs, segmented
        suffix-min down the residual up arcs"""
        zz = self.zz
        A = torch.cummin(ext - zz, -1).values + zz
        key = (A + zz) - BIG * self.sid
        S = torch.flip(torch.cummin(torch.flip(key, [-1]), -1).values, [-1]) + BIG * self.sid - zz
        return torch.clamp(torch.minimum(A, S), max=self.INF)


def column_jacobi(P, max_rounds=100000):
    X, Y, Z = P.seed.shape
    d = torch.full_like(P.seed, P.INF)
    rounds, work, hist = 0, 0, []
    changed_cols = torch.ones((X, Y), dtype=torch.bool, device=d.device)
    while rounds < max_rounds:
        # worklist: columns with a changed neighbour (round 0: all)
        if rounds == 0:
            wl = changed_cols
        else:
            wl = torch.zeros_like(changed_cols)
            for dd in range(4):
                wl |= shift(changed_cols, dd, False)
        nd = P.colsolve(P.ext(d))
        ch = (nd != d).any(-1)
        rounds += 1
        work += int(wl.sum())
        hist.append(int(ch.sum()))
        d = nd
        changed_cols = ch
        if not bool(ch.any()):
            break
    return d, rounds, work, hist


def tile_gs(P, TX, TY, max_rounds=100000):
    X, Y, Z = P.seed.shape
    dev = P.seed.device
    xs = torch.arange(X, device=dev)
    ys = torch.arange(Y, device=dev)
    tx = (xs // TX)[:, None].expand(X, Y)
    ty = (ys // TY)[None, :].expand(X, Y)
    same = []
    for dd in range(4):
        stx, sty = shift(tx, dd, -1), shift(ty, dd, -1)
        same.append(((stx == tx) & (sty == ty))[..., None].expand(X, Y, Z))
    d = torch.full_like(P.seed, P.INF)
    rounds, local_its, tile_work = 0, 0, 0
    ntx, nty = (X + TX - 1) // TX, (Y + TY - 1) // TY
    while rounds < max_rounds:
        frozen = d.clone()
        its = 0
        last = torch.zeros((ntx, nty), dtype=torch.int64, device=dev)  # last local iteration a tile changed
        while True:
            nd = P.colsolve(P.ext(d, frozen, same))
            chc = (nd != d).any(-1)
            d = nd
            its += 1
            if not bool(chc.any()):
                break
            cht = torch.zeros((ntx * TX, nty * TY), dtype=torch.bool, device=dev)
            cht[:X, :Y] = chc
            cht = cht.view(ntx, TX, nty, TY).any(3).any(1)
            last = torch.where(cht, its, last)
        rounds += 1
        local_its += its
        tile_work += int((last + (last > 0)).sum())  # iterations incl. the confirming one, active tiles
        if bool((d == frozen).all()):
            break
    return d, rounds, local_its, tile_work


def main():
    name = sys.argv[1]
    points = [int(s) for s in sys.argv[2].split(",")] if len(sys.argv) > 2 else [64, 256]
    tiles = [(8, 8), (16, 16), (32, 32)]
    spec = V.CONFIGS[name]
    c = torch.from_numpy(V.generate(name)).cuda()
    X, Y, Z = c.shape
    n = X * Y * Z
    INF = n + 1
    for s in points + [0]:
        opts = cg.make_opts(max_sweeps=s if s else 1 << 30)
        h = cg.colgraph_build(c, spec.delta)
        st_, flow, stats = cg.maxflow_solve(h, opts)
        state = torch.empty(8 * n, dtype=torch.int32, device="cuda")
        assert cg.colgraph_export_state(h, state) == 0
        cg.colgraph_free(h)
        P = Problem(state, X, Y, Z, spec.delta, INF)
        torch.cuda.synchronize()
        t0 = time.time()
        d, rounds, work, hist = column_jacobi(P)
        t1 = time.time()
        fin = d[d < INF]
        rec = {"config": name, "max_sweeps": s, "status": st_, "sweeps": stats["sweeps"],
               "relabels": stats["global_relabels"], "bfs_depth": int(fin.max()) if fin.numel() else 0,
               "reachable": int(fin.numel()), "active": int(((P.H >= 0) & (state.view(8, -1)[0].view(X, Y, Z) > 0)).sum()),
               "col_rounds": rounds, "col_work_columns": work, "col_work_over_ncol": work / (X * Y),
               "changed_cols_per_round": hist[:12] + (["..."] + hist[-6:] if len(hist) > 18 else hist[12:]),
               "study_s": round(t1 - t0, 1)}
        if s == 0:  # final state: its H is the library's exact relabel -> must match
            rec["matches_library_bfs"] = bool((torch.clamp(P.H.to(torch.int64), max=INF) == d).all())
        for TX, TY in tiles:
            d2, r2, li, tw = tile_gs(P, TX, TY)
            assert bool((d2 == d).all())
            ntiles = ((X + TX - 1) // TX) * ((Y + TY - 1) // TY)
            rec[f"tile{TX}x{TY}"] = {"rounds": r2, "local_its": li, "tile_its": tw, "tile_its_over_ntiles": tw / ntiles}
        print(json.dumps(rec), flush=True)
        del P, state, d
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
