"""GPU parity for NEXT-4: parallel Boykov-Kolmogorov with hierarchical merging
(§3.1), maxflow_solve_bk, against the CPU oracle bit-exactly -- flow value,
minimal source set (mask) and surface -- on random tiny volumes with random first-stage segment
sizes (1 x 1 columns up to larger than the volume, so zero to many merge stages, ragged edge
segments), general intervals and narrow bands, weight mode, C1/C2 and the C3 golden; the residual
state BK leaves is a maximum flow whose phase-2 export passes the definition checks."""
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


def run_bk(cg, c, delta, seg=(0, 0), weight=False, band=None, export=False):
    t = torch.from_numpy(np.ascontiguousarray(c, np.int32)).cuda()
    if band is not None or (isinstance(delta, (tuple, list)) and len(delta) == 4):
        b = torch.from_numpy(np.ascontiguousarray(band, np.int32)).cuda() if band is not None else None
        h = cg.colgraph_build_general(t, delta, b, None, 0, weight)
    else:
        h = cg.colgraph_build(t, delta, weight)
    try:
        st, flow, stats = cg.maxflow_solve_bk(h, *seg)
        surf = torch.empty(c.shape[:2], dtype=torch.int32, device="cuda")
        mask = torch.empty(c.shape, dtype=torch.uint8, device="cuda")
        est = cg.mincut_extract_surface(h, surf, mask) if st == 0 else -1
        r = {"status": st, "ext": est, "flow": flow, "surface": surf.cpu().numpy(), "mask": mask.cpu().numpy(),
             "stats": stats}
        if export and st == 0:
            est2, F = cg.maxflow_export_flow(h, t, weight)
            r["export_status"], r["F"] = est2, F.cpu().numpy()
        return r
    finally:
        cg.colgraph_free(h)


def same(r, o, ctx, weight=False):
    assert r["status"] == 0, (ctx, r["status"])
    if weight:
        assert r["ext"] == (6 if o["status"] == 6 else 0), ctx
    else:
        assert r["ext"] == 0, (ctx, r["ext"])
    assert r["flow"] == o["flow"], (ctx, r["flow"], o["flow"])
    assert np.array_equal(r["surface"], o["surface"]), ctx
    assert np.array_equal(r["mask"], o["mask"]), ctx


def test_worked_examples(cg):
    ex = json.load(open(os.path.join(GOLDEN_DIR, "worked_examples.json")))["column_examples"]
    for e in ex:
        c = np.array(e["c"], np.int32)
        r = run_bk(cg, c, e["delta"], (1, 1))
        assert r["status"] == 0 and r["ext"] == 0 and r["flow"] == e["flow"], e["name"]
        assert np.array_equal(r["surface"], np.array(e["surface"], np.int32)), e["name"]


def test_random_tiny(cg):
    """600 seeded tiny volumes (tests/.. V.tiny_case) with first-stage segments of 1..6 columns."""
    rng = np.random.default_rng(4242)
    for seed in range(3000, 3600):
        c, delta = V.tiny_case(seed)
        seg = (int(rng.integers(1, 7)), int(rng.integers(1, 7)))
        same(run_bk(cg, c, delta, seg), oracle.colgraph_solve(c, delta), f"seed {seed} {c.shape} d={delta} seg={seg}")


def test_random_larger(cg):
    """Wider volumes (up to 24 x 24 columns, Z up to 70): many merge stages, ragged segments."""
    rng = np.random.default_rng(99)
    for trial in range(60):
        X, Y, Z = int(rng.integers(1, 25)), int(rng.integers(1, 25)), int(rng.integers(1, 71))
        delta = int(rng.integers(0, 6))
        c = rng.integers(0, int(rng.choice([9, 255])) + 1, size=(X, Y, Z)).astype(np.int32)
        seg = (int(rng.integers(1, 9)), int(rng.integers(1, 9)))
        same(run_bk(cg, c, delta, seg), oracle.colgraph_solve(c, delta), f"{trial} {c.shape} d={delta} seg={seg}")


def test_general_intervals_and_bands(cg):
    """NEXT-3 geometry under BK: asymmetric per-direction intervals, narrow bands."""
    from tests.test_gpu_next3 import rand_band, rand_case
    rng = np.random.default_rng(515)
    for k in range(300):
        c, d4 = rand_case(rng)
        seg = (int(rng.integers(1, 4)), int(rng.integers(1, 4)))
        band = rand_band(rng, c, d4) if k % 2 else None
        o = oracle.colgraph_solve(c, d4, band=band)
        same(run_bk(cg, c, d4, seg, band=band), o, f"{k} {c.shape} {d4} band={band is not None}")


def test_weight_mode(cg):
    """Signed vertex weights incl. empty columns (CG_E_EMPTY_COLUMN with the outputs written)."""
    rng = np.random.default_rng(12)
    for trial in range(200):
        X, Y, Z = (int(v) for v in rng.integers(1, 8, 3))
        delta = int(rng.integers(0, 4))
        w = rng.integers(-20, 21, size=(X, Y, Z)).astype(np.int32)
        seg = (int(rng.integers(1, 4)), int(rng.integers(1, 4)))
        o = oracle.colgraph_solve(w, delta, input_is_weight=True)
        same(run_bk(cg, w, delta, seg, weight=True), o, f"{trial} seg={seg}", weight=True)


@pytest.mark.parametrize("seg", [(1, 1), (4, 4), (16, 2), (64, 64)])
def test_c1(cg, seg):
    c = V.generate("C1")
    r = run_bk(cg, c, 2, seg)
    same(r, oracle.colgraph_solve(c, 2), f"C1 seg={seg}")
    # 16 x 16 columns: stages = 1 + number of pairwise merges
    sx, sy = min(seg[0], 16), min(seg[1], 16)
    merges = int(np.ceil(np.log2(16 / sx))) + int(np.ceil(np.log2(16 / sy)))
    assert r["stats"]["bk_stages"] == 1 + merges
    assert r["stats"]["bk_augmentations"] > 0


def test_c2(cg):
    c = V.generate("C2")
    r = run_bk(cg, c, 3)
    same(r, oracle.colgraph_solve(c, 3), "C2")


def test_c3_golden(cg):
    """C3 (16.8 M vertices) against the stored oracle result (scripts/make_oracle_golden.py)."""
    spec = V.CONFIGS["C3"]
    c = V.generate("C3")
    gold = json.load(open(os.path.join(GOLDEN_DIR, "oracle_C3.json")))
    assert gold["input_sha256"] == V.MANIFEST["C3"]
    r = run_bk(cg, c, spec.delta)
    assert r["status"] == 0 and r["ext"] == 0
    assert r["flow"] == gold["flow"]
    assert hashlib.sha256(r["surface"].astype("<i4").tobytes()).hexdigest() == gold["surface_sha256"]
    assert hashlib.sha256(r["mask"].tobytes()).hexdigest() == gold["mask_sha256"]


def test_bk_state_is_a_maximum_flow(cg):
    """The phase-2 export of BK's residual state satisfies Eq. 2/4/5 and its residual cut is the
    oracle's minimal source set (tests/test_gpu_flow.check_flow, independent of the CUDA path)."""
    rng = np.random.default_rng(77)
    for trial in range(120):
        c, delta = V.tiny_case(5000 + trial)
        o = oracle.colgraph_solve(c, delta)
        r = run_bk(cg, c, delta, (int(rng.integers(1, 4)), int(rng.integers(1, 4))), export=True)
        same(r, o, trial)
        assert r["export_status"] == 0, trial
        val, mask = check_flow(c, delta, r["F"])
        assert val == o["flow"], trial
        assert np.array_equal(mask, o["mask"]), trial


def test_errors(cg):
    c = V.generate("C1")
    t = torch.from_numpy(c).cuda()
    h = cg.colgraph_build(t, 2)
    try:
        assert cg.maxflow_solve_bk(h)[0] == 0
        assert cg.maxflow_solve_bk(h)[0] == cg.CG_E_STATE  # already solved
        assert cg.maxflow_solve(h)[0] == cg.CG_E_STATE
    finally:
        cg.colgraph_free(h)
    h = cg.colgraph_build_slabs(t, 2, 2)
    try:
        assert cg.maxflow_solve_bk(h)[0] == cg.CG_E_INVAL  # x-slabs: not supported
    finally:
        cg.colgraph_free(h)
    h = cg.colgraph_build_soft(t, 2, [3, 8])
    try:
        assert cg.maxflow_solve_bk(h)[0] == cg.CG_E_INVAL  # soft arcs: not supported
    finally:
        cg.colgraph_free(h)


def test_time_limit(cg):
    """A stage past its time budget stops with CG_E_NOT_CONVERGED (no hang); 1 ms on C2."""
    c = V.generate("C2")
    t = torch.from_numpy(c).cuda()
    h = cg.colgraph_build(t, 3)
    try:
        st, _, _ = cg.maxflow_solve_bk(h, 128, 128, 1)
        assert st in (cg.CG_E_NOT_CONVERGED, 0)
    finally:
        cg.colgraph_free(h)
