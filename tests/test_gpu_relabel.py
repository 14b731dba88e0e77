"""a2/a5 global relabel: the labels the library leaves are the exact BFS distances to t.

maxflow_solve ends with an exact global relabel (a4; the source-side termination check is switched off
here with CG_SRC_TERM=0), so the heights in the exported state are the
residual-graph distances d(v) to t of the final preflow (§2.1, Alg. 3;
INF = n + 1 for vertices that cannot reach t, reading R8).  The reference here is independent of
the library: the residual graph is rebuilt from the exported flows with scipy and searched from t
(unweighted shortest paths on the reverse graph).  Every relabel flavour is checked: the vertex
BFS over the flag plane (default on one slab), the column fixpoint (default on x-slabs,
CG_RELABEL=colgr; csrc/relabel.cuh) and the record BFS (CG_RELABEL=bfs)."""
import numpy as np
import pytest

from synth import volumes as V

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cg():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_2601_17026_b200 import colgraph
    return colgraph


def exact_labels(state, shape, delta):
    import scipy.sparse as sp
    from scipy.sparse.csgraph import shortest_path
    X, Y, Z = shape
    dx_, dy_ = (delta if isinstance(delta, (tuple, list)) else (delta, delta))
    n = X * Y * Z
    _, _, T, D, L0, L1, L2, L3 = [state[i * n:(i + 1) * n].astype(np.int64).reshape(X, Y, Z) for i in range(8)]
    L = [L0, L1, L2, L3]
    idx = np.arange(n).reshape(X, Y, Z)
    zs = np.arange(Z)
    rows, cols = [], []
    tnode = n
    m = T > 0
    rows.append(idx[m]); cols.append(np.full(int(m.sum()), tnode))                 # v -> t
    rows.append(idx[:, :, 1:].ravel()); cols.append(idx[:, :, :-1].ravel())      # down, INF
    m = D[:, :, 1:] > 0
    rows.append(idx[:, :, :-1][m]); cols.append(idx[:, :, 1:][m])                 # up, residual D(z+1)
    for d, (dx, dy) in enumerate([(1, 0), (-1, 0), (0, 1), (0, -1)]):
        dl = dx_ if d < 2 else dy_
        zo = np.where(zs == 0, 0, np.where(zs > dl, zs - dl, -1))
        xs = slice(max(0, -dx), X - max(0, dx)); xt = slice(max(0, dx), X - max(0, -dx))
        ys = slice(max(0, -dy), Y - max(0, dy)); yt = slice(max(0, dy), Y - max(0, -dy))
        valid = np.flatnonzero(zo >= 0)
        tail = idx[xs, ys][:, :, valid]
        head = idx[xt, yt][:, :, zo[valid]]
        rows.append(tail.ravel()); cols.append(head.ravel())                       # lateral, INF
        m = L[d][xs, ys][:, :, valid] > 0
        rows.append(head[m]); cols.append(tail[m])                                 # its reverse, residual L
    r = np.concatenate(rows); cl = np.concatenate(cols)
    rev = sp.csr_matrix((np.ones(len(r), np.int8), (cl, r)), shape=(n + 1, n + 1))
    dist = shortest_path(rev, directed=True, unweighted=True, indices=tnode)[:n]
    return np.where(np.isinf(dist), n + 1, dist).astype(np.int64)


def solve_state(cg, c, delta, nslabs=1, weight=False):
    t = torch.from_numpy(np.ascontiguousarray(c, np.int32)).cuda()
    h = cg.colgraph_build(t, delta, weight) if nslabs == 1 else cg.colgraph_build_slabs(t, delta, nslabs, weight)
    try:
        st, flow, stats = cg.maxflow_solve(h, None)
        assert st == 0
        out = torch.empty(8 * c.size, dtype=torch.int32, device="cuda")
        assert cg.colgraph_export_state(h, out) == 0
        return out.cpu().numpy(), stats
    finally:
        cg.colgraph_free(h)


@pytest.fixture(params=["default", "flags", "colgr", "bfs", "trunc", "trunc_sticky", "trunc_off", "bottomup", "dense_all",
                        "dense_off"])
def flavour(request, monkeypatch):
    # the labels are exact after an exhaustive relabel: end every solve on one (no source-side check)
    monkeypatch.setenv("CG_SRC_TERM", "0")
    if request.param == "default":
        monkeypatch.delenv("CG_RELABEL", raising=False)
    elif request.param == "trunc":  # truncated relabels mid-solve; the last one is exhaustive
        monkeypatch.delenv("CG_RELABEL", raising=False)
        monkeypatch.setenv("CG_BFS_TRUNC", "64,2")
    elif request.param == "trunc_sticky":  # truncation also after the first quiescent batch (third field 0)
        monkeypatch.delenv("CG_RELABEL", raising=False)
        monkeypatch.setenv("CG_BFS_TRUNC", "64,2,0")
    elif request.param == "trunc_off":  # every relabel exhaustive (the default truncates: 65536,32)
        monkeypatch.delenv("CG_RELABEL", raising=False)
        monkeypatch.setenv("CG_BFS_TRUNC", "0,0")
    elif request.param in ("dense_all", "dense_off"):  # dense bit-plane levels for every level / never
        monkeypatch.delenv("CG_RELABEL", raising=False)
        monkeypatch.setenv("CG_BFS_DENSE", "1" if request.param == "dense_all" else "0")
    elif request.param == "bottomup":  # flag-plane BFS with bottom-up levels whenever allowed
        monkeypatch.delenv("CG_RELABEL", raising=False)
        monkeypatch.setenv("CG_BFS_BU", "1000000,1")
    else:
        monkeypatch.setenv("CG_RELABEL", request.param)
    return request.param


def check(cg, c, delta, nslabs=1, weight=False, ctx=""):
    state, stats = solve_state(cg, c, delta, nslabs, weight)
    n = c.size
    H = state[n:2 * n].astype(np.int64)
    ref = exact_labels(state, c.shape, delta)
    bad = np.flatnonzero(H != ref)
    assert bad.size == 0, (ctx, bad[:5], H[bad[:5]], ref[bad[:5]])
    return stats


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_labels_exact_configs(cg, flavour, name):
    spec = V.CONFIGS[name]
    check(cg, V.generate(name), spec.delta, ctx=name)


def test_labels_exact_random_tiny(cg, flavour):
    for seed in range(6000, 6150):
        c, delta = V.tiny_case(seed)
        check(cg, c, delta, ctx=f"seed {seed}")


def test_labels_exact_weight_mode(cg, flavour):
    rng = np.random.default_rng(21)
    for k in range(60):
        X, Y, Z = int(rng.integers(1, 6)), int(rng.integers(1, 6)), int(rng.integers(1, 40))
        w = rng.integers(-20, 21, size=(X, Y, Z)).astype(np.int32)
        check(cg, w, int(rng.integers(0, 4)), weight=True, ctx=f"w{k}")


def test_labels_exact_anisotropic(cg, flavour):
    rng = np.random.default_rng(22)
    for k in range(40):
        X, Y, Z = int(rng.integers(1, 7)), int(rng.integers(1, 7)), int(rng.integers(2, 70))
        c = rng.integers(0, 50, size=(X, Y, Z)).astype(np.int32)
        check(cg, c, (int(rng.integers(0, 5)), int(rng.integers(0, 5))), ctx=f"a{k}")


def test_labels_exact_tall_columns(cg, flavour):
    """Z spans several chunks with ragged tails (Z = 33, 97, 255, 256) and the > 256 fallback."""
    rng = np.random.default_rng(23)
    for Z in (33, 97, 200, 255, 256, 300):
        c = rng.integers(0, 255, size=(3, 4, Z)).astype(np.int32)
        check(cg, c, 3, ctx=f"Z{Z}")


@pytest.mark.parametrize("ns", [2, 3, 5])
def test_labels_exact_slabs(cg, flavour, ns):
    c = V.generate("C2")[:40]
    check(cg, c, 3, nslabs=ns, ctx=f"C2 crop /{ns}")


@pytest.mark.parametrize("each", ["0", "1"])
def test_labels_exact_slabs_bfs_launch(cg, monkeypatch, each):
    """In-process slabs: the in-slab BFS of all slabs in one launch (default) or one launch per slab."""
    monkeypatch.delenv("CG_RELABEL", raising=False)
    monkeypatch.setenv("CG_SLAB_BFS_EACH", each)
    for ns in (2, 4, 7):
        check(cg, V.generate("C2")[:56], 3, nslabs=ns, ctx=f"C2 crop /{ns} each={each}")


def test_colgr_counts_rounds(cg, monkeypatch):
    """The fixpoint reports its rounds in gr_passes (one launch per relabel on one slab)."""
    monkeypatch.setenv("CG_RELABEL", "colgr")
    c = V.generate("C2")
    _, stats = solve_state(cg, c, 3)
    assert stats["gr_passes"] >= stats["global_relabels"] > 0


@pytest.mark.parametrize("dense", ["1", "5", "40", "0"])
def test_labels_exact_dense_levels(cg, monkeypatch, dense):
    """Dense bit-plane BFS levels (kernels.cuh bfs_dense_level; one slab, Z % 32 == 0): columns of one
    to four 32-z words, intervals 0..31 on either axis (and 32, which the host routes to the list
    levels), thresholds from "every level" to "never"; the labels equal the scipy distances."""
    monkeypatch.delenv("CG_RELABEL", raising=False)
    monkeypatch.setenv("CG_SRC_TERM", "0")
    monkeypatch.setenv("CG_BFS_DENSE", dense)
    rng = np.random.default_rng(31)
    for k in range(40):
        X, Y, Z = int(rng.integers(1, 7)), int(rng.integers(1, 7)), 32 * int(rng.integers(1, 5))
        cmax = int(rng.choice([3, 9, 255]))
        c = rng.integers(0, cmax + 1, size=(X, Y, Z)).astype(np.int32)
        dl = (int(rng.choice([0, 1, 2, 4, 7, 31, 32])), int(rng.choice([0, 1, 3, 16, 31])))
        check(cg, c, dl if k % 2 else dl[0], ctx=f"d{k} {X}x{Y}x{Z} {dl}")
