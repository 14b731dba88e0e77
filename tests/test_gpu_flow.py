"""NEXT-2: phase 2 + flow export.  maxflow_export_flow must return a
maximum FLOW on the Wu-Chen arcs.  Checked against the definitions, independently of the
CUDA path: capacity (Eq. 2), conservation at every vertex (Eq. 4), value
= the oracle's |f| (Eq. 5), and the cut read off the flow's residual graph (BFS from s,
Theorem 1) = the oracle's minimal source set."""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import breadth_first_order

import oracle
from synth import volumes as V

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

DIRS = [(1, 0), (-1, 0), (0, 1), (0, -1)]


@pytest.fixture(scope="module")
def cg():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_2601_17026_b200 import colgraph
    return colgraph


def weights(c, weight, band=None):
    cc = c.astype(np.int64)
    if weight:
        return cc
    w = np.empty_like(cc)
    if band is not None:  # narrow band (reading R15): base rule inside [lo, hi), no terminal arc outside
        w[:] = 0
        X, Y, _ = c.shape
        for x in range(X):
            for y in range(Y):
                lo, hi = int(band[x, y, 0]), int(band[x, y, 1])
                w[x, y, lo] = cc[x, y, lo] - (cc[x, y, lo:hi].sum() + 1)
                w[x, y, lo + 1:hi] = cc[x, y, lo + 1:hi] - cc[x, y, lo:hi - 1]
        return w
    w[:, :, 0] = cc[:, :, 0] - (cc.sum(axis=2) + 1)
    w[:, :, 1:] = cc[:, :, 1:] - cc[:, :, :-1]
    return w


def d4_of(delta):
    if isinstance(delta, (tuple, list)):
        if len(delta) == 4:
            return tuple(int(v) for v in delta)
        return (int(delta[0]), int(delta[0]), int(delta[1]), int(delta[1]))
    return (int(delta),) * 4


def sl(dx, X):  # (source slice, target slice) along one axis for a shift dx
    return slice(max(0, -dx), X - max(0, dx)), slice(max(0, dx), X - max(0, -dx))


def soft_caps(penalty):
    f = [0] + [int(v) for v in penalty]
    return [f[1]] + [f[k + 1] - 2 * f[k] + f[k - 1] for k in range(1, len(penalty))]


def check_flow(c, delta, F, weight=False, penalty=None, band=None):
    X, Y, Z = c.shape
    n = X * Y * Z
    fs, ft, fd, *L = [F[i].astype(np.int64) for i in range(7)]
    d4 = d4_of(delta)  # edge interval of each vertex's lateral arc toward +x, -x, +y, -y
    K = max(d4) if penalty is not None else 0  # the library's soft arcs per direction
    caps = soft_caps(penalty)[:K] if K else []
    w = weights(c, weight, band)
    E0, T0 = np.maximum(-w, 0), np.maximum(w, 0)
    zs = np.arange(Z)
    ZO = [np.where(zs == 0, 0, np.where(zs > dl, zs - dl, -1)) for dl in d4]  # per direction
    # Eq. 2: capacities (infinite arcs: non-negative); arcs that do not exist carry nothing
    assert (fs >= 0).all() and (fs <= E0).all()
    assert (ft >= 0).all() and (ft <= T0).all()
    assert (fd >= 0).all() and (fd[:, :, 0] == 0).all()
    for d, (dx, dy) in enumerate(DIRS):
        valid = ZO[d] >= 0
        assert (L[d] >= 0).all() and (L[d][:, :, ~valid] == 0).all()
        if dx == 1: assert (L[d][X - 1] == 0).all()
        if dx == -1: assert (L[d][0] == 0).all()
        if dy == 1: assert (L[d][:, Y - 1] == 0).all()
        if dy == -1: assert (L[d][:, 0] == 0).all()
    SF = {}
    for d in range(4 if K else 0):
        for k in range(K):
            f = F[7 + d * K + k].astype(np.int64)
            SF[d, k] = f
            dx, dy = DIRS[d]
            exists = np.zeros((X, Y, Z), bool)
            if k < d4[d] and caps[k] > 0:
                xs, _ = sl(dx, X)
                ys, _ = sl(dy, Y)
                exists[xs, ys, k:] = True
            assert (f >= 0).all() and (f <= (caps[k] if caps else 0)).all(), (d, k)
            assert (f[~exists] == 0).all(), (d, k)
    # Eq. 4: conservation at every vertex
    net = fs - ft - fd
    net[:, :, :-1] += fd[:, :, 1:]
    for d, (dx, dy) in enumerate(DIRS):
        zo = ZO[d]
        valid = zo >= 0
        net -= L[d]
        xs, xt = sl(dx, X)
        ys, yt = sl(dy, Y)
        src = L[d][xs, ys][:, :, valid]
        tgt = net[xt, yt]
        for k, z in enumerate(zs[valid]):
            tgt[:, :, zo[z]] += src[:, :, k]
    for (d, k), f in SF.items():
        dx, dy = DIRS[d]
        xs, xt = sl(dx, X)
        ys, yt = sl(dy, Y)
        net -= f
        if Z - k > 0:
            net[xt, yt, :Z - k] += f[xs, ys, k:]
    assert not net.any(), "conservation violated"
    assert ft.sum() == fs.sum()
    # residual graph of the flow; BFS from s
    idx = np.arange(n).reshape(X, Y, Z)
    s_node, t_node = n, n + 1
    rows, cols = [], []
    m = fs < E0
    rows.append(np.full(m.sum(), s_node)); cols.append(idx[m])
    m = ft < T0
    rows.append(idx[m]); cols.append(np.full(m.sum(), t_node))
    rows.append(idx[:, :, 1:].ravel()); cols.append(idx[:, :, :-1].ravel())
    m = fd[:, :, 1:] > 0
    rows.append(idx[:, :, :-1][m]); cols.append(idx[:, :, 1:][m])
    for d, (dx, dy) in enumerate(DIRS):
        zo = ZO[d]
        xs, xt = sl(dx, X)
        ys, yt = sl(dy, Y)
        vz = np.flatnonzero(zo >= 0)
        tail = idx[xs, ys][:, :, vz]
        head = idx[xt, yt][:, :, zo[vz]]
        rows.append(tail.ravel()); cols.append(head.ravel())
        m = L[d][xs, ys][:, :, vz] > 0
        rows.append(head[m]); cols.append(tail[m])
    for (d, k), f in SF.items():
        if Z - k <= 0:
            continue
        dx, dy = DIRS[d]
        xs, xt = sl(dx, X)
        ys, yt = sl(dy, Y)
        tail = idx[xs, ys][:, :, k:]
        head = idx[xt, yt][:, :, :Z - k]
        fk = f[xs, ys][:, :, k:]
        m = fk < caps[k]
        rows.append(tail[m]); cols.append(head[m])
        m = fk > 0
        rows.append(head[m]); cols.append(tail[m])
    r = np.concatenate(rows); cl = np.concatenate(cols)
    g = sp.csr_matrix((np.ones(len(r), np.int8), (r, cl)), shape=(n + 2, n + 2))
    reach = breadth_first_order(g, s_node, directed=True, return_predecessors=False)
    assert t_node not in set(reach.tolist()), "augmenting path left"
    mask = np.zeros(n, np.uint8)
    mask[reach[reach < n]] = 1
    return int(ft.sum()), mask.reshape(X, Y, Z)


def export(cg, c, delta, weight=False, opts=None, extract_first=True, penalty=None):
    t = torch.from_numpy(np.ascontiguousarray(c, np.int32)).cuda()
    h = cg.colgraph_build_soft(t, delta, penalty, weight) if penalty is not None else cg.colgraph_build(t, delta, weight)
    try:
        st, flow, _ = cg.maxflow_solve(h, None)
        assert st == 0
        if extract_first:
            surf = torch.empty(c.shape[:2], dtype=torch.int32, device="cuda")
            assert cg.mincut_extract_surface(h, surf) in (0, 6)
        dxy0 = tuple(delta) if isinstance(delta, (tuple, list)) else (delta, delta)
        st, F = cg.maxflow_export_flow(h, t, weight, opts=opts, soft_k=max(dxy0) if penalty is not None else 0)
        assert st == 0, cg.STATUS.get(st)
        if extract_first:
            surf2 = torch.empty(c.shape[:2], dtype=torch.int32, device="cuda")
            assert cg.mincut_extract_surface(h, surf2) == cg.CG_E_STATE
            assert cg.maxflow_export_flow(h, t, weight)[0] == cg.CG_E_STATE
        return flow, F.cpu().numpy()
    finally:
        cg.colgraph_free(h)


def test_flow_random_tiny(cg):
    for seed in range(1000, 1300):
        c, delta = V.tiny_case(seed)
        o = oracle.colgraph_solve(c, delta)
        flow, F = export(cg, c, delta)
        val, mask = check_flow(c, delta, F)
        assert flow == val == o["flow"], seed
        assert np.array_equal(mask, o["mask"]), seed


def test_flow_weight_mode(cg):
    rng = np.random.default_rng(5)
    for trial in range(100):
        X, Y, Z = (int(v) for v in rng.integers(1, 7, 3))
        delta = int(rng.integers(0, 4))
        w = rng.integers(-20, 21, size=(X, Y, Z)).astype(np.int32)
        o = oracle.colgraph_solve(w, delta, input_is_weight=True)
        flow, F = export(cg, w, delta, weight=True)
        val, mask = check_flow(w, delta, F, weight=True)
        assert flow == val == o["flow"], trial
        assert np.array_equal(mask, o["mask"]), trial


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_flow_configs(cg, name):
    c = V.generate(name)
    delta = V.CONFIGS[name].delta
    o = oracle.colgraph_solve(c, delta)
    flow, F = export(cg, c, delta, extract_first=False)
    val, mask = check_flow(c, delta, F)
    assert flow == val == o["flow"]
    assert np.array_equal(mask, o["mask"])


def test_flow_slabs(cg):
    """Phase 2 + export on in-process x-slabs (the NCCL path's messages): whole-volume output."""
    rng = np.random.default_rng(9)
    for trial in range(150):
        c, delta = V.tiny_case(2000 + trial)
        if c.shape[0] < 2:
            continue
        ns = 2 + trial % min(3, c.shape[0] - 1)
        pen = [int(v) for v in np.cumsum(np.sort(rng.integers(0, 9, max(delta, 1))))] if trial % 3 == 0 else None
        K = delta if pen is not None else 0
        t = torch.from_numpy(np.ascontiguousarray(c)).cuda()
        h = cg.colgraph_build_slabs_soft(t, delta, pen, ns) if pen is not None else cg.colgraph_build_slabs(t, delta, ns)
        try:
            st, flow, _ = cg.maxflow_solve(h, None)
            assert st == 0
            st, F = cg.maxflow_export_flow(h, t, soft_k=K)
            assert st == 0, (trial, cg.STATUS.get(st))
        finally:
            cg.colgraph_free(h)
        o = oracle.colgraph_solve(c, delta, penalty=pen)
        val, mask = check_flow(c, delta, F.cpu().numpy(), penalty=pen)
        assert flow == val == o["flow"] and np.array_equal(mask, o["mask"]), (trial, ns, pen)


def test_flow_errors(cg):
    t = torch.zeros((2, 2, 3), dtype=torch.int32, device="cuda")
    h = cg.colgraph_build(t, 1)
    try:
        assert cg.maxflow_export_flow(h, t)[0] == cg.CG_E_STATE  # not solved yet
    finally:
        cg.colgraph_free(h)



def test_flow_generic_phase2(cg, monkeypatch):
    """The generic phase 2 (push-relabel toward s; the fallback after capped same-level
    cancellation) gives a valid maximum flow too."""
    monkeypatch.setenv("CG_PHASE2_PR", "1")
    for seed in range(1000, 1100):
        c, delta = V.tiny_case(seed)
        o = oracle.colgraph_solve(c, delta)
        flow, F = export(cg, c, delta)
        val, mask = check_flow(c, delta, F)
        assert flow == val == o["flow"] and np.array_equal(mask, o["mask"]), seed
