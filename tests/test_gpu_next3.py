"""GPU parity for the rest of NEXT-3: general (asymmetric) edge intervals toward
+x/-x/+y/-y and narrow bands (reading R15), through
colgraph_build_general, against the oracle bit-exactly (flow value, minimal source set, surface) on
every flavour: one slab, in-process x-slabs, loopback NCCL ranks, tiles, soft smoothness and the
phase-2 flow export (checked against the definitions, tests/test_gpu_flow.check_flow)."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from synth import volumes as V
from tests import pins
from tests.test_gpu_flow import check_flow

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
GOLDEN_DIR = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def cg():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_2601_17026_b200 import colgraph
    return colgraph


def run(cg, c, d4, band=None, nslabs=1, penalty=None, opts=None):
    t = torch.from_numpy(np.ascontiguousarray(c, np.int32)).cuda()
    b = torch.from_numpy(np.ascontiguousarray(band, np.int32)).cuda() if band is not None else None
    h = cg.colgraph_build_general(t, d4, b, penalty, nslabs if nslabs > 1 else 0)
    try:
        st, flow, _ = cg.maxflow_solve(h, opts)
        surf = torch.empty(c.shape[:2], dtype=torch.int32, device="cuda")
        mask = torch.empty(c.shape, dtype=torch.uint8, device="cuda")
        est = cg.mincut_extract_surface(h, surf, mask) if st == 0 else -1
        return {"status": st, "ext": est, "flow": flow, "surface": surf.cpu().numpy(), "mask": mask.cpu().numpy()}
    finally:
        cg.colgraph_free(h)


def same(r, o, ctx):
    assert r["status"] == 0 and r["ext"] == 0, (ctx, r["status"], r["ext"])
    assert r["flow"] == o["flow"], (ctx, r["flow"], o["flow"])
    assert np.array_equal(r["surface"], o["surface"]), ctx
    assert np.array_equal(r["mask"], o["mask"]), ctx


def rand_case(rng, zmax=12):
    X, Y, Z = int(rng.integers(1, 6)), int(rng.integers(1, 6)), int(rng.integers(1, zmax))
    c = rng.integers(0, int(rng.choice([3, 9, 255])) + 1, size=(X, Y, Z)).astype(np.int32)
    d4 = tuple(int(v) for v in rng.integers(0, 5, size=4))
    return c, d4


def rand_band(rng, c, d4):
    X, Y, Z = c.shape
    for _ in range(100):
        lo = rng.integers(0, Z, size=(X, Y))
        hi = np.minimum(lo + rng.integers(1, Z + 1, size=(X, Y)), Z)
        band = np.stack([lo, hi], axis=-1).astype(np.int32)
        if pins.band_consistent(band, d4):
            return band
    band = np.zeros((X, Y, 2), np.int32)
    band[..., 1] = Z
    return band


def test_asymmetric_random(cg):
    rng = np.random.default_rng(8100)
    for k in range(400):
        c, d4 = rand_case(rng)
        same(run(cg, c, d4), oracle.colgraph_solve(c, d4), f"{k} {c.shape} {d4}")


def test_asymmetric_taller_columns(cg):
    """Several chunks per column with ragged tails; intervals up to 40."""
    rng = np.random.default_rng(8150)
    for k in range(40):
        X, Y, Z = int(rng.integers(1, 5)), int(rng.integers(1, 5)), int(rng.integers(30, 140))
        c = rng.integers(0, 255, size=(X, Y, Z)).astype(np.int32)
        d4 = tuple(int(v) for v in rng.integers(0, 41, size=4))
        same(run(cg, c, d4), oracle.colgraph_solve(c, d4), f"tall {k} {c.shape} {d4}")


def test_band_random(cg):
    rng = np.random.default_rng(8200)
    for k in range(300):
        c, d4 = rand_case(rng)
        if k % 3 == 0:
            d4 = (d4[0],) * 4
        band = rand_band(rng, c, d4)
        o = oracle.colgraph_solve(c, d4, band=band)
        same(run(cg, c, d4, band), o, f"{k} {c.shape} {d4} {band.tolist()}")


def test_band_inconsistent_is_still_the_weighted_cut(cg):
    """Bands that move faster than the intervals: the result is still the minimal cut of the band
    weights (oracle), only its reading as a banded surface needs the precondition."""
    rng = np.random.default_rng(8250)
    for k in range(100):
        c, d4 = rand_case(rng)
        X, Y, Z = c.shape
        lo = rng.integers(0, Z, size=(X, Y))
        band = np.stack([lo, np.minimum(lo + rng.integers(1, Z + 1, size=(X, Y)), Z)], -1).astype(np.int32)
        o = oracle.colgraph_solve(c, d4, band=band)
        r = run(cg, c, d4, band)
        assert r["flow"] == o["flow"] and np.array_equal(r["mask"], o["mask"]), k


@pytest.mark.parametrize("ns", [2, 3])
def test_next3_slabs(cg, ns):
    rng = np.random.default_rng(8300 + ns)
    done = 0
    for k in range(150):
        c, d4 = rand_case(rng)
        if c.shape[0] < ns:
            continue
        band = rand_band(rng, c, d4) if k % 2 else None
        same(run(cg, c, d4, band, nslabs=ns), oracle.colgraph_solve(c, d4, band=band), f"{k} {d4} /{ns}")
        done += 1
    assert done > 50


def test_next3_tiles(cg):
    rng = np.random.default_rng(8400)
    opts = cg.make_opts(sweep_kind=cg.SWEEP_TILES)
    for k in range(60):
        c, d4 = rand_case(rng)
        band = rand_band(rng, c, d4) if k % 2 else None
        same(run(cg, c, d4, band, opts=opts), oracle.colgraph_solve(c, d4, band=band), f"tiles {k} {d4}")


def test_next3_soft(cg):
    rng = np.random.default_rng(8500)
    for k in range(150):
        c, d4 = rand_case(rng, zmax=9)
        K = max(max(d4), 1)
        pen = [int(v) for v in np.cumsum(np.cumsum(rng.integers(0, 4, size=K)))]
        band = rand_band(rng, c, d4) if k % 2 else None
        same(run(cg, c, d4, band, penalty=pen), oracle.colgraph_solve(c, d4, penalty=pen, band=band),
             f"soft {k} {d4} {pen}")


def test_next3_ranks(cg):
    from tests.test_gpu_nccl_loopback import solve_ranks  # noqa: F401  (same helper, general builder)
    cg.nccl_loopback(True)
    try:
        import threading
        rng = np.random.default_rng(8600)
        for k in range(25):
            c, d4 = rand_case(rng)
            X, Y, Z = c.shape
            if X < 2:
                continue
            band = rand_band(rng, c, d4) if k % 2 else None
            R = int(rng.integers(2, min(X, 4) + 1))
            nid = cg.nccl_unique_id()
            dims = cg.cg_dims(X, Y, Z, d4[0], d4[2])
            out = [None] * R
            errs = []

            def rank_main(r):
                try:
                    x0, x1 = cg.cg_slab_range(X, Y, Z, 0, r, R)
                    t = torch.from_numpy(c[x0:x1].copy()).cuda()
                    b = torch.from_numpy(band[x0:x1].copy()).cuda() if band is not None else None
                    s = torch.cuda.Stream()
                    h = cg.colgraph_build_general(t, d4, b, None, 0, stream=s, rank=r, nranks=R, nccl_id=nid,
                                                  dims=dims)
                    try:
                        st, flow, _ = cg.maxflow_solve(h)
                        with torch.cuda.stream(s):
                            surf = torch.empty((x1 - x0, Y), dtype=torch.int32, device="cuda")
                        est = cg.mincut_extract_surface(h, surf)
                        s.synchronize()
                        out[r] = (st, est, flow, surf.cpu().numpy())
                    finally:
                        cg.colgraph_free(h)
                except Exception as e:  # noqa: BLE001
                    errs.append(e)

            th = [threading.Thread(target=rank_main, args=(r,)) for r in range(R)]
            [t.start() for t in th]
            [t.join(timeout=300) for t in th]
            assert not errs, errs
            o = oracle.colgraph_solve(c, d4, band=band)
            assert all(x[0] == 0 and x[1] == 0 and x[2] == o["flow"] for x in out), k
            assert np.array_equal(np.concatenate([x[3] for x in out], 0), o["surface"]), k
    finally:
        cg.nccl_loopback(False)


def test_next3_flow_export(cg):
    rng = np.random.default_rng(8700)
    for k in range(100):
        c, d4 = rand_case(rng)
        band = rand_band(rng, c, d4) if k % 2 else None
        t = torch.from_numpy(c).cuda()
        b = torch.from_numpy(band).cuda() if band is not None else None
        h = cg.colgraph_build_general(t, d4, b, None, 0)
        try:
            st, flow, _ = cg.maxflow_solve(h)
            assert st == 0
            st, F = cg.maxflow_export_flow(h, t)
            assert st == 0
        finally:
            cg.colgraph_free(h)
        o = oracle.colgraph_solve(c, d4, band=band)
        val, mask = check_flow(c, d4, F.cpu().numpy(), band=band)
        assert val == o["flow"] == flow and np.array_equal(mask, o["mask"]), k


def test_band_rejections(cg):
    c = torch.zeros((2, 3, 6), dtype=torch.int32, device="cuda")
    bad = torch.zeros((2, 3, 2), dtype=torch.int32, device="cuda")  # lo == hi
    with pytest.raises(cg.ColgraphError):
        cg.colgraph_build_general(c, 1, bad)
    ok = torch.zeros((2, 3, 2), dtype=torch.int32, device="cuda")
    ok[..., 1] = 6
    with pytest.raises(cg.ColgraphError):
        cg.colgraph_build_general(c, 1, ok, input_is_weight=True)
    with pytest.raises(cg.ColgraphError):
        cg.colgraph_build_general(c, (1, -1, 1, 1))


@pytest.mark.parametrize("name,half", [("C2", 8), ("C4", 12)])
def test_band_around_the_optimum(cg, name, half):
    """A narrow band of +-half around the (unbanded) optimal surface -- the paper's landmark-band
    setting -- keeps that surface: the lowest optimum lies in the band, and the band only removes
    other candidates.  C2 against a live oracle, C4 (the headline config) against its stored result."""
    spec = V.CONFIGS[name]
    c = V.generate(name)
    if name == "C2":
        ref = oracle.colgraph_solve(c, spec.delta, want_mask=False)["surface"]
    else:
        gfile = os.path.join(GOLDEN_DIR, f"oracle_{name}_surface.npz")
        ref = np.load(gfile)["surface"]
    Z = spec.Z
    band = np.stack([np.maximum(ref - half, 0), np.minimum(ref + half + 1, Z)], -1).astype(np.int32)
    assert pins.band_consistent(band, spec.delta)
    r = run(cg, c, spec.delta, band)
    assert r["status"] == 0 and r["ext"] == 0
    assert np.array_equal(r["surface"], ref)
    if name == "C4":
        gold = json.load(open(os.path.join(GOLDEN_DIR, "oracle_C4.json")))
        assert hashlib.sha256(r["surface"].astype("<i4").tobytes()).hexdigest() == gold["surface_sha256"]
    # value: cost of the surface + the band constant (weak duality with the feasible banded surface)
    assert r["flow"] == pins.surface_cost(c, r["surface"]) + pins.k0_band(c, band)
