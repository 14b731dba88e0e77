"""Edge cases at the limits of the ABI (GPU): the largest volume colgraph_build accepts
(n = X*Y*Z just under 2^31, ~105 GB of device memory) and degenerate dimensions.

At the size limit the expected values come from a closed form: with
costs that depend on z only, every column is the same line, the optimal surface is flat at
the LOWEST argmin of c(z) (any Delta), and
    |f| = min cost + K0 = X*Y * (min_z c(z) + sum_{z>=1} max(0, c(z-1) - c(z)) - c(0)).
Every column carries flow (c(z) has several drops), so the walks, the relabel and the
extraction all index vertices up to 2^31 - 1."""
import numpy as np
import pytest

import oracle
from tests.test_gpu_parity import gpu

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cg():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_2601_17026_b200 import colgraph
    return colgraph


PROFILE = np.array([200, 120, 180, 90, 140, 60, 110, 160, 70, 150, 30, 130, 210, 40, 90, 250,
                    80, 120, 20, 170, 100, 60, 140, 200, 50, 90, 180, 110, 70, 160, 120, 190], np.int64)


def closed_form(X, Y, c):
    drops = np.maximum(0, c[:-1] - c[1:]).sum()
    return X * Y * int(c.min() + drops - c[0]), int(np.argmin(c))


def test_profile_closed_form_small(cg):
    """The closed form itself, checked against the oracle on a small volume."""
    X, Y = 5, 4
    c = np.broadcast_to(PROFILE.astype(np.int32), (X, Y, PROFILE.size)).copy()
    flow, zstar = closed_form(X, Y, PROFILE)
    o = oracle.colgraph_solve(c, 2)
    assert o["flow"] == flow and (o["surface"] == zstar).all()
    r = gpu(cg, c, 2)
    assert r["flow"] == flow and (r["surface"] == zstar).all()


def test_largest_volume(cg):
    free, _ = torch.cuda.mem_get_info()
    X, Y, Z = 65520, 1024, PROFILE.size  # n = 2,146,959,360 < INT32_MAX - Z - 64
    n = X * Y * Z
    need = n * (4 + 32 + 12) + (1 << 30)
    if free < need:
        pytest.skip(f"needs {need / 2**30:.0f} GiB of device memory, {free / 2**30:.0f} free")
    cost = torch.from_numpy(PROFILE.astype(np.int32)).cuda().expand(X, Y, Z).contiguous()
    flow, zstar = closed_form(X, Y, PROFILE)
    h = cg.colgraph_build(cost, 3)
    try:
        del cost
        torch.cuda.empty_cache()
        st, f, stats = cg.maxflow_solve(h, None)
        assert st == cg.CG_OK and f == flow, (st, f, flow)
        surf = torch.empty((X, Y), dtype=torch.int32, device="cuda")
        assert cg.mincut_extract_surface(h, surf) == cg.CG_OK
        assert int(surf.min()) == zstar == int(surf.max())
    finally:
        cg.colgraph_free(h)


def test_size_limit_rejected(cg):
    t = torch.zeros((1, 1, 1), dtype=torch.int32, device="cuda")
    for dims in [(65536, 1024, 32), (1 << 16, 1 << 15, 2)]:  # n >= 2^31 - Z - 64
        d = cg.cg_dims(*dims, 1)
        import ctypes
        h = ctypes.c_void_p()
        st = cg.lib().colgraph_build(ctypes.byref(d), ctypes.c_void_p(t.data_ptr()), 0, None, ctypes.byref(h))
        assert st == cg.CG_E_INVAL, dims


@pytest.mark.parametrize("dims", [(0, 4, 4), (4, 0, 4), (4, 4, 0)])
def test_empty_dims_rejected(cg, dims):
    import ctypes
    t = torch.zeros((1, 1, 1), dtype=torch.int32, device="cuda")
    d = cg.cg_dims(*dims, 1)
    h = ctypes.c_void_p()
    assert cg.lib().colgraph_build(ctypes.byref(d), ctypes.c_void_p(t.data_ptr()), 0, None, ctypes.byref(h)) == cg.CG_E_INVAL
