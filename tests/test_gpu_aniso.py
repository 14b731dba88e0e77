"""NEXT-3: anisotropic smoothness Delta_x != Delta_y (the edge interval is
defined per adjacent column).  GPU results through the C ABI vs the CPU oracle,
bit-exact, on every solver flavour: vertex walks, x-slabs, tiles, and the phase-2 flow."""
import numpy as np
import pytest

import oracle
from synth import volumes as V
from tests.test_gpu_flow import check_flow, export
from tests.test_gpu_parity import assert_same, gpu

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cg():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_2601_17026_b200 import colgraph
    return colgraph


def cases(n, seed):
    rng = np.random.default_rng(seed)
    for _ in range(n):
        X, Y, Z = int(rng.integers(1, 7)), int(rng.integers(1, 7)), int(rng.integers(1, 14))
        dxy = (int(rng.integers(0, 5)), int(rng.integers(0, 5)))
        cmax = (4, 10, 256)[int(rng.integers(0, 3))]
        yield rng.integers(0, cmax, size=(X, Y, Z)).astype(np.int32), dxy


def test_aniso_random_tiny(cg):
    for i, (c, dxy) in enumerate(cases(400, 41)):
        assert_same(gpu(cg, c, dxy), oracle.colgraph_solve(c, dxy), f"case {i} {c.shape} {dxy}")


@pytest.mark.parametrize("dxy", [(1, 3), (3, 1), (0, 2), (4, 0)])
def test_aniso_c1(cg, dxy):
    c = V.generate("C1")
    assert_same(gpu(cg, c, dxy), oracle.colgraph_solve(c, dxy), str(dxy))


def test_aniso_c2(cg):
    c = V.generate("C2")
    assert_same(gpu(cg, c, (2, 5)), oracle.colgraph_solve(c, (2, 5)))


def test_aniso_slabs(cg):
    for i, (c, dxy) in enumerate(cases(150, 42)):
        if c.shape[0] < 2:
            continue
        ns = int(1 + i % min(4, c.shape[0]))
        t = torch.from_numpy(c).cuda()
        r = cg.solve(t, dxy, nslabs=ns)
        o = oracle.colgraph_solve(c, dxy)
        assert r["flow"] == o["flow"], (i, ns)
        assert np.array_equal(r["mask"].cpu().numpy(), o["mask"]), (i, ns)


def test_aniso_tiles(cg):
    opts = cg.make_opts(sweep_kind=cg.SWEEP_TILES)
    for i, (c, dxy) in enumerate(cases(200, 43)):
        assert_same(gpu(cg, c, dxy, opts=opts), oracle.colgraph_solve(c, dxy), f"case {i}")


def test_aniso_flow_export(cg):
    for i, (c, dxy) in enumerate(cases(100, 44)):
        o = oracle.colgraph_solve(c, dxy)
        flow, F = export(cg, c, dxy)
        val, mask = check_flow(c, dxy, F)
        assert flow == val == o["flow"] and np.array_equal(mask, o["mask"]), i


def test_isotropic_default_unchanged(cg):
    c = V.generate("C1")
    a, b = gpu(cg, c, 2), gpu(cg, c, (2, 2))
    assert a["flow"] == b["flow"] and np.array_equal(a["mask"], b["mask"])
    t = torch.zeros((2, 2, 3), dtype=torch.int32, device="cuda")
    with pytest.raises(cg.ColgraphError):
        cg.colgraph_build(t, (1, -2))
