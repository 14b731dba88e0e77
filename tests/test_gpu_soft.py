"""NEXT-1: soft smoothness -- the VCE-weight net surface problem of
PAPER.md:42-43 (convex edge costs over the edge interval).  GPU (colgraph_build_soft) vs the
CPU oracle built with the same penalty, bit-exact on |f|, minimal source set and surface,
across solver schedules; the oracle itself is pinned by brute force in tests/test_oracle.py."""
import numpy as np
import pytest

import oracle
from synth import volumes as V
from tests.test_gpu_parity import assert_same

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cg():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_2601_17026_b200 import colgraph
    return colgraph


def convex(rng, K):
    return np.cumsum(np.sort(rng.integers(0, 12, K))).astype(np.int32)


def gpu_soft(cg, c, delta, pen, weight=False, opts=None):
    t = torch.from_numpy(np.ascontiguousarray(c, np.int32)).cuda()
    r = cg.solve(t, delta, weight, True, opts, penalty=pen)
    r["surface"] = r["surface"].cpu().numpy()
    r["mask"] = r["mask"].cpu().numpy()
    return r


def cases(n, seed):
    rng = np.random.default_rng(seed)
    for _ in range(n):
        X, Y, Z = int(rng.integers(1, 7)), int(rng.integers(1, 7)), int(rng.integers(1, 14))
        dxy = (int(rng.integers(0, 5)), int(rng.integers(0, 5)))
        pen = convex(rng, max(dxy[0], dxy[1], 1))
        cmax = (4, 10, 256)[int(rng.integers(0, 3))]
        yield rng.integers(0, cmax, size=(X, Y, Z)).astype(np.int32), dxy, pen


def test_soft_random_tiny(cg):
    for i, (c, dxy, pen) in enumerate(cases(400, 61)):
        o = oracle.colgraph_solve(c, dxy, penalty=pen)
        assert_same(gpu_soft(cg, c, dxy, pen), o, f"case {i} {c.shape} {dxy} {pen}")


@pytest.mark.parametrize("opts", [dict(walk_len=-1), dict(walk_len=3), dict(check_every=1, gr_factor=0.25)])
def test_soft_schedules(cg, opts):
    for i, (c, dxy, pen) in enumerate(cases(100, 62)):
        o = oracle.colgraph_solve(c, dxy, penalty=pen)
        assert_same(gpu_soft(cg, c, dxy, pen, opts=cg.make_opts(**opts)), o, f"{opts} case {i}")


@pytest.mark.parametrize("var", [{"CG_BFS_LEVEL_LAUNCHES": "1"}, {"CG_WALK_MIN": "0"}])
def test_soft_variants(cg, monkeypatch, var):
    for k, v in var.items():
        monkeypatch.setenv(k, v)
    for i, (c, dxy, pen) in enumerate(cases(100, 63)):
        assert_same(gpu_soft(cg, c, dxy, pen), oracle.colgraph_solve(c, dxy, penalty=pen), f"{var} case {i}")


def test_soft_weight_mode(cg):
    rng = np.random.default_rng(64)
    for trial in range(100):
        X, Y, Z = (int(v) for v in rng.integers(1, 7, 3))
        delta = int(rng.integers(0, 4))
        pen = convex(rng, max(delta, 1))
        w = rng.integers(-20, 21, size=(X, Y, Z)).astype(np.int32)
        o = oracle.colgraph_solve(w, delta, input_is_weight=True, penalty=pen)
        r = gpu_soft(cg, w, delta, pen, weight=True)
        assert r["flow"] == o["flow"] and np.array_equal(r["mask"], o["mask"]), trial


@pytest.mark.parametrize("name,pen", [("C1", [3, 8]), ("C1", [0, 40]), ("C2", [5, 12, 25])])
def test_soft_configs(cg, name, pen):
    c = V.generate(name)
    delta = V.CONFIGS[name].delta
    o = oracle.colgraph_solve(c, delta, penalty=pen)
    assert_same(gpu_soft(cg, c, delta, pen), o, name)


def test_soft_errors(cg):
    t = torch.zeros((3, 3, 5), dtype=torch.int32, device="cuda")
    for pen in ([5, 6], [1]):  # non-convex; shorter than Delta = 2
        with pytest.raises(cg.ColgraphError) as e:
            cg.colgraph_build_soft(t, 2, pen)
        assert e.value.status == cg.CG_E_INVAL
    h = cg.colgraph_build_soft(t, 2, [1, 3])
    try:
        assert cg.maxflow_solve(h, cg.make_opts(sweep_kind=cg.SWEEP_TILES))[0] == cg.CG_E_INVAL
        assert cg.maxflow_solve(h, None)[0] == 0
    finally:
        cg.colgraph_free(h)


def test_soft_full_size_c3(cg):
    """C3 (16.8 M vertices) with a soft penalty: |f| = sum c(S) + sum_pairs f(|dS|) + K0 for the
    returned Delta-feasible surface -- the cut of that surface equals the flow, which proves
    both optimal (weak duality); the mask is {z <= S}."""
    from tests import pins
    spec = V.CONFIGS["C3"]
    c = V.generate("C3")
    pen = [4, 11]
    r = gpu_soft(cg, c, spec.delta, pen)
    s = r["surface"]
    assert r["status"] == 0 and r["extract_status"] == 0
    dsx, dsy = np.abs(np.diff(s.astype(np.int64), axis=0)), np.abs(np.diff(s.astype(np.int64), axis=1))
    assert max(dsx.max(), dsy.max()) <= spec.delta
    f = np.array([0] + pen, np.int64)
    assert r["flow"] == pins.surface_cost(c, s) + int(f[dsx].sum() + f[dsy].sum()) + pins.k0(c)
    assert np.array_equal(r["mask"].sum(axis=2) - 1, s)


def test_soft_slabs_random(cg):
    """x-slabs (in-process transport: the NCCL path's messages, device copies) with soft arcs."""
    for i, (c, dxy, pen) in enumerate(cases(250, 65)):
        if c.shape[0] < 2:
            continue
        ns = 2 + i % min(3, c.shape[0] - 1)
        t = torch.from_numpy(c).cuda()
        r = cg.solve(t, dxy, penalty=pen, nslabs=ns)
        o = oracle.colgraph_solve(c, dxy, penalty=pen)
        assert r["status"] == 0, (i, r["status"])
        assert r["flow"] == o["flow"], (i, ns, c.shape, dxy, pen)
        assert np.array_equal(r["mask"].cpu().numpy(), o["mask"]), (i, ns)


@pytest.mark.parametrize("name,ns,pen", [("C1", 3, [3, 8]), ("C2", 4, [5, 12, 25])])
def test_soft_slabs_configs(cg, name, ns, pen):
    c = V.generate(name)
    delta = V.CONFIGS[name].delta
    o = oracle.colgraph_solve(c, delta, penalty=pen)
    r = cg.solve(torch.from_numpy(c).cuda(), delta, penalty=pen, nslabs=ns)
    assert r["flow"] == o["flow"] and np.array_equal(r["mask"].cpu().numpy(), o["mask"])


def test_soft_flow_export(cg, monkeypatch):
    """NEXT-1 x NEXT-2: the maximum flow of a soft graph, checked against the definitions
    (capacities incl. soft arcs, conservation, value = oracle, residual cut = oracle mask)."""
    from tests.test_gpu_flow import check_flow, export
    for i, (c, dxy, pen) in enumerate(cases(150, 66)):
        K = max(dxy[0], dxy[1], 1)
        pen = list(pen[:K]) + [int(pen[-1])] * (K - len(pen))
        o = oracle.colgraph_solve(c, dxy, penalty=pen)
        flow, F = export(cg, c, dxy, penalty=pen)
        val, mask = check_flow(c, dxy, F, penalty=pen)
        assert flow == val == o["flow"] and np.array_equal(mask, o["mask"]), i
    monkeypatch.setenv("CG_PHASE2_PR", "1")  # the generic phase 2 on soft graphs
    for i, (c, dxy, pen) in enumerate(cases(60, 67)):
        o = oracle.colgraph_solve(c, dxy, penalty=pen)
        flow, F = export(cg, c, dxy, penalty=list(pen))
        val, mask = check_flow(c, dxy, F, penalty=list(pen))
        assert flow == val == o["flow"] and np.array_equal(mask, o["mask"]), i
