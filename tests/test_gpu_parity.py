"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit-exact
on |f|, the minimal source set and the surface (integer work,
so the bar is exact equality).  Full-size configs without a stored oracle
result are checked through properties that hold at any size."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from synth import volumes as V
from tests import pins

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
GOLDEN_DIR = os.path.join(os.path.dirname(__file__), "golden")
WORKED = json.load(open(os.path.join(GOLDEN_DIR, "worked_examples.json")))


@pytest.fixture(scope="module")
def cg():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_2601_17026_b200 import colgraph
    return colgraph


def gpu(cg, c, delta, weight=False, opts=None, mask=True):
    t = torch.from_numpy(np.ascontiguousarray(c, np.int32)).cuda()
    r = cg.solve(t, delta, weight, mask, opts)
    r["surface"] = r["surface"].cpu().numpy()
    r["mask"] = r["mask"].cpu().numpy() if r["mask"] is not None else None
    return r


def assert_same(r, o, ctx=""):
    assert r["status"] == 0, (ctx, r["status"])
    assert r["flow"] == o["flow"], (ctx, r["flow"], o["flow"])
    assert np.array_equal(r["surface"], o["surface"]), ctx
    if r["mask"] is not None and o["mask"] is not None:
        assert np.array_equal(r["mask"], o["mask"]), ctx


# ---------------------------------------------------------------- small exact cases

@pytest.mark.parametrize("ex", WORKED["column_examples"], ids=lambda e: e["name"])
def test_worked_examples(cg, ex):
    c = np.array(ex["c"], np.int32)
    r = gpu(cg, c, ex["delta"])
    assert r["status"] == 0 and r["extract_status"] == 0
    assert r["flow"] == ex["flow"]
    assert np.array_equal(r["surface"], np.array(ex["surface"], np.int32))


def test_random_tiny_sweep(cg):
    """1000 seeded tiny volumes (X, Y <= 5, Z <= 12, Delta 0..4, cost ranges 3/9/255)."""
    for seed in range(1000, 2000):
        c, delta = V.tiny_case(seed)
        o = oracle.colgraph_solve(c, delta)
        r = gpu(cg, c, delta)
        assert r["extract_status"] == 0, seed
        assert_same(r, o, f"seed {seed} shape {c.shape} delta {delta}")


def test_weight_mode_random(cg):
    """Signed vertex weights (input_is_weight=1), incl. empty columns -> CG_E_EMPTY_COLUMN."""
    rng = np.random.default_rng(11)
    for trial in range(200):
        X, Y, Z = (int(v) for v in rng.integers(1, 7, 3))
        delta = int(rng.integers(0, 4))
        w = rng.integers(-20, 21, size=(X, Y, Z)).astype(np.int32)
        o = oracle.colgraph_solve(w, delta, input_is_weight=True)
        r = gpu(cg, w, delta, weight=True)
        assert r["status"] == 0
        assert r["flow"] == o["flow"], trial
        assert np.array_equal(r["surface"], o["surface"]), trial
        assert np.array_equal(r["mask"], o["mask"]), trial
        assert r["extract_status"] == (6 if o["status"] == 6 else 0), trial


@pytest.mark.parametrize("shape,delta", [((1, 1, 1), 0), ((1, 1, 40), 3), ((37, 1, 9), 1), ((1, 29, 70), 2),
                                         ((6, 7, 33), 0), ((5, 4, 65), 64), ((9, 3, 31), 40), ((3, 3, 100), 1)])
def test_edge_shapes(cg, shape, delta):
    """Ragged z tails (Z not a multiple of 32), X=1 / Y=1, Delta=0 and Delta >= Z-1."""
    c = V.tiny(500 + sum(shape) + delta, *shape, 255)
    o = oracle.colgraph_solve(c, delta)
    assert_same(gpu(cg, c, delta), o, str(shape))


def test_constant_costs(cg):
    c = np.full((5, 6, 7), 17, np.int32)
    o = oracle.colgraph_solve(c, 1)
    assert_same(gpu(cg, c, 1), o)


# ---------------------------------------------------------------- configs

def test_c1(cg):
    c = V.generate("C1")
    o = oracle.colgraph_solve(c, 2)
    r = gpu(cg, c, 2)
    assert_same(r, o, "C1")


def test_c2(cg):
    c = V.generate("C2")
    assert V.sha256_volume(c) == V.MANIFEST["C2"]
    o = oracle.colgraph_solve(c, 3)
    r = gpu(cg, c, 3)
    assert_same(r, o, "C2")


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_full_size(cg, name):
    """Bench launch configuration (default options).  Exact comparison against the
    stored oracle result (scripts/make_oracle_golden.py) when present; always the
    properties: |f| = cost(surface) + K0 with a Delta-feasible surface (which proves
    both optimal by weak duality), mask = {z <= surface}."""
    spec = V.CONFIGS[name]
    c = V.generate(name)
    assert V.sha256_volume(c) == V.MANIFEST[name]
    r = gpu(cg, c, spec.delta, mask=True)
    assert r["status"] == 0 and r["extract_status"] == 0
    s = r["surface"]
    assert np.abs(np.diff(s.astype(np.int64), axis=0)).max() <= spec.delta
    assert np.abs(np.diff(s.astype(np.int64), axis=1)).max() <= spec.delta
    assert r["flow"] == pins.surface_cost(c, s) + pins.k0(c)
    Z = spec.Z
    tops = r["mask"].sum(axis=2) - 1
    assert np.array_equal(tops, s)
    gfile = os.path.join(GOLDEN_DIR, f"oracle_{name}.json")
    if os.path.exists(gfile):
        gold = json.load(open(gfile))
        assert gold["input_sha256"] == V.MANIFEST[name]
        assert r["flow"] == gold["flow"]
        assert hashlib.sha256(s.astype("<i4").tobytes()).hexdigest() == gold["surface_sha256"]
        assert hashlib.sha256(r["mask"].tobytes()).hexdigest() == gold["mask_sha256"]


# ---------------------------------------------------------------- certificate, determinism, options, API

def _certificate(c, delta, state):
    """Independent O(n) certificate on the exported SoA: residuals >= 0, exact
    conservation (Eq. 4 with excess, Eq. 8), and no residual path from a vertex with
    excess to t (so the preflow is maximum)."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import breadth_first_order
    X, Y, Z = c.shape
    n = X * Y * Z
    E, H, T, D, L0, L1, L2, L3 = [state[i * n:(i + 1) * n].astype(np.int64).reshape(X, Y, Z) for i in range(8)]
    L = [L0, L1, L2, L3]
    cc = c.astype(np.int64)
    w = np.empty_like(cc)
    w[:, :, 0] = cc[:, :, 0] - (cc.sum(axis=2) + 1)
    w[:, :, 1:] = cc[:, :, 1:] - cc[:, :, :-1]
    E0, T0 = np.maximum(-w, 0), np.maximum(w, 0)
    assert (E >= 0).all() and (T >= 0).all() and (T <= T0).all() and (D >= 0).all()
    assert all((l >= 0).all() for l in L)
    assert (D[:, :, 0] == 0).all()
    zs = np.arange(Z)
    zo = np.where(zs == 0, 0, np.where(zs > delta, zs - delta, -1))
    # conservation: E = E0 - (T0 - T) - D + D(z+1) - sum_d L_d + lateral inflow
    net = E0 - (T0 - T) - D
    net[:, :, :-1] += D[:, :, 1:]
    dirs = [(1, 0), (-1, 0), (0, 1), (0, -1)]
    for d, (dx, dy) in enumerate(dirs):
        net -= L[d]
        xs = slice(max(0, -dx), X - max(0, dx))
        xt = slice(max(0, dx), X - max(0, -dx))
        ys = slice(max(0, -dy), Y - max(0, dy))
        yt = slice(max(0, dy), Y - max(0, -dy))
        valid = zo >= 0
        src = L[d][xs, ys][:, :, valid]
        tgt = net[xt, yt]
        for k, z in enumerate(zs[valid]):
            tgt[:, :, zo[z]] += src[:, :, k]
        # flow on lateral arcs whose tail has no neighbour must be 0
        if dx == 1: assert (L[d][X - 1] == 0).all()
        if dx == -1: assert (L[d][0] == 0).all()
        if dy == 1: assert (L[d][:, Y - 1] == 0).all()
        if dy == -1: assert (L[d][:, 0] == 0).all()
        assert (L[d][:, :, ~valid] == 0).all()
    assert np.array_equal(net, E), "conservation violated"
    # residual graph (forward arcs: u -> v with residual > 0), then BFS from t on the reverse graph
    idx = np.arange(n).reshape(X, Y, Z)
    rows, cols = [], []
    tnode = n
    m = T > 0
    rows.append(idx[m]); cols.append(np.full(m.sum(), tnode))
    rows.append(idx[:, :, 1:].ravel()); cols.append(idx[:, :, :-1].ravel())      # down, INF
    m = D[:, :, 1:] > 0
    rows.append(idx[:, :, :-1][m]); cols.append(idx[:, :, 1:][m])                 # up, residual D(z+1)
    for d, (dx, dy) in enumerate(dirs):
        xs = slice(max(0, -dx), X - max(0, dx)); xt = slice(max(0, dx), X - max(0, -dx))
        ys = slice(max(0, -dy), Y - max(0, dy)); yt = slice(max(0, dy), Y - max(0, -dy))
        valid = np.flatnonzero(zo >= 0)
        tail = idx[xs, ys][:, :, valid]
        head = idx[xt, yt][:, :, zo[valid]]
        rows.append(tail.ravel()); cols.append(head.ravel())                       # lateral, INF
        m = L[d][xs, ys][:, :, valid] > 0
        rows.append(head[m]); cols.append(tail[m])                                 # reverse, residual L
    r = np.concatenate(rows); cl = np.concatenate(cols)
    rev = sp.csr_matrix((np.ones(len(r), np.int8), (cl, r)), shape=(n + 1, n + 1))
    reach = breadth_first_order(rev, tnode, directed=True, return_predecessors=False)
    reach = reach[reach < n]
    assert not (E.ravel()[reach] > 0).any(), "a vertex with excess can still reach t"


def test_certificate_c2(cg):
    c = V.generate("C2")
    t = torch.from_numpy(c).cuda()
    h = cg.colgraph_build(t, 3)
    try:
        st, flow, stats = cg.maxflow_solve(h, None)
        assert st == 0
        out = torch.empty(8 * c.size, dtype=torch.int32, device="cuda")
        assert cg.colgraph_export_state(h, out) == 0
        state = out.cpu().numpy()
    finally:
        cg.colgraph_free(h)
    _certificate(c, 3, state)
    T0 = np.maximum(np.diff(c.astype(np.int64), axis=2), 0).sum()
    T = state[2 * c.size:3 * c.size].astype(np.int64).sum()
    assert flow == T0 - T


def test_determinism(cg):
    """100 solves of C2 (lock-free schedules differ run to run): the value, surface and minimal
    source set must not (SURVEY.md §4 item 6 stress)."""
    c = V.generate("C2")
    o = oracle.colgraph_solve(c, 3)
    key0 = (o["flow"], hashlib.sha256(o["surface"].tobytes()).hexdigest(), hashlib.sha256(o["mask"].tobytes()).hexdigest())
    works = set()
    for _ in range(100):
        r = gpu(cg, c, 3)
        key = (r["flow"], hashlib.sha256(r["surface"].tobytes()).hexdigest(),
               hashlib.sha256(r["mask"].tobytes()).hexdigest())
        assert key == key0
        works.add(r["stats"]["work"])
    assert len(works) > 1  # the schedules really differed


def test_source_side_termination(cg, monkeypatch):
    """a4 by the source side: a quiescent solve may end when the residual closure of the vertices with
    excess reaches no arc into t (csrc/colgraph.cu source_side_done) instead of on an exhaustive
    relabel; the extraction then reuses that closure.  Both ways give the oracle's result, and the
    check does end solves (src_terminated) -- also when capped to one batch of rounds."""
    ended = 0
    for cap in ("48", "16", "0"):
        monkeypatch.setenv("CG_SRC_TERM", cap)
        for seed in range(1000, 1200):
            c, delta = V.tiny_case(seed)
            r = gpu(cg, c, delta)
            assert_same(r, oracle.colgraph_solve(c, delta), f"cap {cap} seed {seed}")
            if cap == "0":
                assert r["stats"]["src_terminated"] == 0
            else:
                ended += r["stats"]["src_terminated"]
        for name, delta in (("C1", 2), ("C2", 3)):
            c = V.generate(name)
            r = gpu(cg, c, delta)
            assert_same(r, oracle.colgraph_solve(c, delta), f"cap {cap} {name}")
            ended += r["stats"]["src_terminated"] if cap != "0" else 0
    assert ended > 100


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_certificate_full_size(cg, name):
    """The O(n) max-preflow certificate (capacities, exact conservation, no residual path from excess
    to t) on the exported state of a full-size solve in the bench's launch configuration."""
    spec = V.CONFIGS[name]
    c = V.generate(name)
    t = torch.from_numpy(c).cuda()
    h = cg.colgraph_build(t, spec.delta)
    try:
        st, flow, stats = cg.maxflow_solve(h, None)
        assert st == 0
        out = torch.empty(8 * c.size, dtype=torch.int32, device="cuda")
        assert cg.colgraph_export_state(h, out) == 0
        state = out.cpu().numpy()
    finally:
        cg.colgraph_free(h)
    del t
    _certificate(c, spec.delta, state)


@pytest.mark.parametrize("kw", [dict(gap_every=4), dict(ops_per_sweep=4), dict(gr_factor=0.25),
                                dict(gr_factor=2.0, check_every=1), dict(gap_every=1, ops_per_sweep=2),
                                dict(walk_len=-1), dict(walk_len=1), dict(walk_len=7), dict(walk_len=4096)])
@pytest.mark.parametrize("name", ["C1", "C2"])
def test_options_do_not_change_results(cg, kw, name):
    c = V.generate(name)
    delta = V.CONFIGS[name].delta
    o = oracle.colgraph_solve(c, delta)
    assert_same(gpu(cg, c, delta, opts=cg.make_opts(**kw)), o, str(kw))


def test_host_api_matches_device_api(cg):
    c = V.generate("C2")
    a = cg.colgraph_solve_host(c, 3, want_mask=True)
    b = gpu(cg, c, 3)
    assert a["status"] == 0 and a["flow"] == b["flow"]
    assert np.array_equal(a["surface"], b["surface"]) and np.array_equal(a["mask"], b["mask"])


def test_metamorphic_gpu(cg):
    c = V.generate("C1")
    base = gpu(cg, c, 2)
    fx = gpu(cg, c[::-1].copy(), 2)
    assert fx["flow"] == base["flow"] and np.array_equal(fx["surface"], base["surface"][::-1])
    tr = gpu(cg, np.ascontiguousarray(c.transpose(1, 0, 2)), 2)
    assert tr["flow"] == base["flow"] and np.array_equal(tr["surface"], base["surface"].T)
    plus = gpu(cg, c + 11, 2)
    assert plus["flow"] == base["flow"] and np.array_equal(plus["surface"], base["surface"])


def test_error_paths(cg):
    t = torch.zeros((2, 2, 2), dtype=torch.int32, device="cuda")
    with pytest.raises(cg.ColgraphError) as e:
        cg.colgraph_build(t, -1)
    assert e.value.status == cg.CG_E_INVAL
    w = torch.tensor([[[-2**31, 5]]], dtype=torch.int32, device="cuda")
    with pytest.raises(cg.ColgraphError) as e:
        cg.colgraph_build(w, 1, input_is_weight=True)
    assert e.value.status == cg.CG_E_OVERFLOW
    h = cg.colgraph_build(t, 1)
    try:
        surf = torch.empty((2, 2), dtype=torch.int32, device="cuda")
        assert cg.mincut_extract_surface(h, surf) == cg.CG_E_STATE
        st, flow, _ = cg.maxflow_solve(h, None)
        assert st == 0
        assert cg.maxflow_solve(h, None)[0] == cg.CG_E_STATE
    finally:
        cg.colgraph_free(h)


def test_not_converged_status(cg):
    c = V.generate("C2")
    t = torch.from_numpy(c).cuda()
    h = cg.colgraph_build(t, 3)
    try:
        st, _, _ = cg.maxflow_solve(h, cg.make_opts(max_sweeps=1, check_every=1))
        assert st == cg.CG_E_NOT_CONVERGED
    finally:
        cg.colgraph_free(h)
