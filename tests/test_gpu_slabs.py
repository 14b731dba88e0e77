"""x-slab (multi-GPU) algorithm, run as several slabs in one process on one GPU
(colgraph_build_slabs: the same halo messages as the NCCL ranks, moved with
device-to-device copies).  Results must be bit-identical to the oracle and to the
single-slab solve (unique by §8(c) c3, so any difference is a bug)."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from synth import volumes as V

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
GOLDEN_DIR = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def cg():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_2601_17026_b200 import colgraph
    return colgraph


def run(cg, c, delta, nslabs, weight=False, opts=None):
    t = torch.from_numpy(np.ascontiguousarray(c, np.int32)).cuda()
    r = cg.solve(t, delta, weight, True, opts, nslabs=nslabs)
    r["surface"] = r["surface"].cpu().numpy()
    r["mask"] = r["mask"].cpu().numpy()
    return r


def same(r, o, ctx):
    assert r["status"] == 0, ctx
    assert r["flow"] == o["flow"], (ctx, r["flow"], o["flow"])
    assert np.array_equal(r["surface"], o["surface"]), ctx
    assert np.array_equal(r["mask"], o["mask"]), ctx


def test_random_tiny_slabs(cg):
    rng = np.random.default_rng(5)
    for seed in range(3000, 3300):
        c, delta = V.tiny_case(seed)
        X = c.shape[0]
        if X < 2:
            continue
        ns = int(rng.integers(2, X + 1))
        o = oracle.colgraph_solve(c, delta)
        same(run(cg, c, delta, ns), o, f"seed {seed} shape {c.shape} delta {delta} slabs {ns}")


@pytest.mark.parametrize("ns", [2, 3, 7, 16])
def test_c1_slabs(cg, ns):
    c = V.generate("C1")
    same(run(cg, c, 2, ns), oracle.colgraph_solve(c, 2), f"C1/{ns}")


@pytest.mark.parametrize("ns", [2, 4, 8])
def test_c2_slabs(cg, ns):
    c = V.generate("C2")
    same(run(cg, c, 3, ns), oracle.colgraph_solve(c, 3), f"C2/{ns}")


@pytest.mark.parametrize("kw", [dict(walk_len=-1), dict(walk_len=3), dict(check_every=1)])
def test_slab_options(cg, kw):
    c = V.generate("C2")[:, :64]
    c = np.ascontiguousarray(c)
    same(run(cg, c, 3, 4, opts=cg.make_opts(**kw)), oracle.colgraph_solve(c, 3), str(kw))


def test_weight_mode_slabs(cg):
    rng = np.random.default_rng(17)
    for trial in range(60):
        X, Y, Z = int(rng.integers(2, 8)), int(rng.integers(1, 6)), int(rng.integers(1, 7))
        delta = int(rng.integers(0, 3))
        w = rng.integers(-20, 21, size=(X, Y, Z)).astype(np.int32)
        o = oracle.colgraph_solve(w, delta, input_is_weight=True)
        r = run(cg, w, delta, int(rng.integers(2, X + 1)), weight=True)
        assert r["flow"] == o["flow"] and np.array_equal(r["surface"], o["surface"]), trial
        assert r["extract_status"] == (6 if o["status"] == 6 else 0), trial


@pytest.mark.parametrize("name,ns", [("C3", 2), ("C3", 5), ("C4", 8), ("C5", 4)])
def test_full_size_slabs(cg, name, ns):
    spec = V.CONFIGS[name]
    gfile = os.path.join(GOLDEN_DIR, f"oracle_{name}.json")
    if not os.path.exists(gfile):
        pytest.skip("no stored oracle result")
    gold = json.load(open(gfile))
    r = run(cg, V.generate(name), spec.delta, ns)
    assert r["status"] == 0 and r["flow"] == gold["flow"]
    assert hashlib.sha256(r["surface"].astype("<i4").tobytes()).hexdigest() == gold["surface_sha256"]
    assert hashlib.sha256(r["mask"].tobytes()).hexdigest() == gold["mask_sha256"]


def test_slab_state_export_is_a_max_preflow(cg):
    """Whole-volume export of a 4-slab solve passes the same O(n) certificate as 1 slab."""
    from tests.test_gpu_parity import _certificate
    c = V.generate("C2")
    t = torch.from_numpy(c).cuda()
    h = cg.colgraph_build_slabs(t, 3, 4)
    try:
        st, flow, _ = cg.maxflow_solve(h, None)
        assert st == 0
        out = torch.empty(8 * c.size, dtype=torch.int32, device="cuda")
        assert cg.colgraph_export_state(h, out) == 0
        state = out.cpu().numpy()
    finally:
        cg.colgraph_free(h)
    _certificate(c, 3, state)


def test_bfs_slab_relabel(cg, monkeypatch):
    """The level-synchronous vertex-BFS x-slab relabel (CG_RELABEL=bfs), the alternative to the
    default column fixpoint with boundary exchanges, must give the same unique results."""
    monkeypatch.setenv("CG_RELABEL", "bfs")
    for seed in range(3000, 3060):
        c, delta = V.tiny_case(seed)
        ns = 2 + seed % 4
        if c.shape[0] < ns:
            continue
        same(run(cg, c, delta, ns), oracle.colgraph_solve(c, delta), f"seed {seed} slabs {ns}")
    c = V.generate("C1")
    o = oracle.colgraph_solve(c, V.CONFIGS["C1"].delta)
    for ns in (2, 3):
        same(run(cg, c, V.CONFIGS["C1"].delta, ns), o, f"C1 x{ns}")