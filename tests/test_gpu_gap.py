"""a5 gap heuristic (§2.1; the paper left parallel gap relabeling open, L534).

With the relabel triggers pushed far out (gr_factor and the time trigger CG_GR_BETA large), vertices
cut off from t climb between relabels and gaps open in the label histogram; gap_every = 1 runs the
heuristic after every sweep batch.  These tests require that it actually lifts vertices
(gap_lifted > 0 -- a stubbed k_gap_lift fails them) and that results stay bit-exact, on one slab,
on in-process x-slabs (summed histograms) and on loopback NCCL ranks (allreduced histograms)."""
import os

import numpy as np
import pytest

import oracle
from synth import volumes as V

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cg():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_2601_17026_b200 import colgraph
    return colgraph


@pytest.fixture
def rare_relabels(monkeypatch):
    monkeypatch.setenv("CG_GR_BETA", "1000")


def run(cg, c, delta, nslabs=1, **kw):
    t = torch.from_numpy(np.ascontiguousarray(c, np.int32)).cuda()
    r = cg.solve(t, delta, False, True, cg.make_opts(**kw), nslabs=nslabs)
    r["surface"] = r["surface"].cpu().numpy()
    r["mask"] = r["mask"].cpu().numpy()
    return r


def same(r, o, ctx):
    assert r["status"] == 0 and r["extract_status"] == 0, ctx
    assert r["flow"] == o["flow"], (ctx, r["flow"], o["flow"])
    assert np.array_equal(r["surface"], o["surface"]), ctx
    assert np.array_equal(r["mask"], o["mask"]), ctx


GAP = dict(gap_every=1, gr_factor=1000.0, check_every=1)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_gap_lifts_and_stays_exact(cg, rare_relabels, name):
    spec = V.CONFIGS[name]
    c = V.generate(name)
    r = run(cg, c, spec.delta, **GAP)
    same(r, oracle.colgraph_solve(c, spec.delta), name)
    assert r["stats"]["gap_runs"] > 0
    assert r["stats"]["gap_lifted"] > 0, r["stats"]


@pytest.mark.parametrize("ns", [2, 3])
def test_gap_on_slabs(cg, rare_relabels, ns):
    c = V.generate("C2")
    r = run(cg, c, 3, nslabs=ns, **GAP)
    same(r, oracle.colgraph_solve(c, 3), f"C2/{ns}")
    assert r["stats"]["gap_lifted"] > 0, r["stats"]


def test_gap_random_tiny(cg, rare_relabels):
    lifted = 0
    for seed in range(5000, 5150):
        c, delta = V.tiny_case(seed)
        r = run(cg, c, delta, **GAP)
        same(r, oracle.colgraph_solve(c, delta), f"seed {seed}")
        lifted += r["stats"]["gap_lifted"]
    assert lifted > 0


def test_gap_loopback_ranks(cg, rare_relabels):
    from tests.test_gpu_nccl_loopback import solve_ranks
    cg.nccl_loopback(True)
    try:
        c = V.generate("C2")
        r = solve_ranks(cg, c, 3, 3, opts=cg.make_opts(**GAP))
    finally:
        cg.nccl_loopback(False)
    same({**r, "extract_status": r["ext"]}, oracle.colgraph_solve(c, 3), "C2 ranks")
    assert sum(o["stats"]["gap_lifted"] for o in r["ranks"]) > 0
