"""GPU parity of the alternative a3/a2 implementations against the CPU oracle (bit-exact):
  - CG_SWEEP_TILES: checkerboard tile discharge in shared memory (tile.cuh), incl. ragged
    tiles (X, Y not multiples of the tile shape) and every instantiated lane segment S;
  - the vertex-frontier BFS relabel (CG_RELABEL=bfs) vs the default column fixpoint, and
    within it the level-per-launch BFS (CG_BFS_LEVEL_LAUNCHES=1) vs the persistent one;
  - the sweep/relabel knobs of include/colgraph.h: a replayed relabel schedule
    (CG_GR_SCHEDULE), work-only trigger, single hops only, small-worklist thresholds.
The options change the schedule only; the max-flow value, the minimal source set and the
surface are unique, so results must be identical."""
import os

import numpy as np
import pytest

import oracle
from synth import volumes as V
from tests.test_gpu_parity import assert_same, gpu

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def cg():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_2601_17026_b200 import colgraph
    return colgraph


@pytest.fixture
def env(monkeypatch):
    return monkeypatch


def tiles(cg, **kw):
    return cg.make_opts(sweep_kind=cg.SWEEP_TILES, **kw)


def test_tiles_random_tiny(cg):
    for seed in range(1000, 1400):
        c, delta = V.tiny_case(seed)
        o = oracle.colgraph_solve(c, delta)
        assert_same(gpu(cg, c, delta, opts=tiles(cg)), o, f"seed {seed}")


# Z picks the lane segment S in {1, 2, 3, 4, 6, 8}; X, Y ragged against 4x4 tiles
@pytest.mark.parametrize("shape,delta", [((5, 7, 9), 1), ((9, 6, 33), 2), ((7, 5, 70), 3), ((6, 9, 100), 1),
                                         ((5, 5, 150), 4), ((3, 6, 256), 2), ((1, 1, 40), 0), ((13, 1, 20), 1)])
def test_tiles_shapes(cg, shape, delta):
    c = V.tiny(900 + sum(shape) + delta, *shape, 255)
    o = oracle.colgraph_solve(c, delta)
    assert_same(gpu(cg, c, delta, opts=tiles(cg)), o, str(shape))


@pytest.mark.parametrize("kw", [dict(), dict(tile_steps=1), dict(tile_steps=3, tile_relabel_every=-1),
                                dict(tile_relabel_every=1), dict(check_every=1)])
@pytest.mark.parametrize("name", ["C1", "C2"])
def test_tiles_configs(cg, kw, name):
    c = V.generate(name)
    delta = V.CONFIGS[name].delta
    o = oracle.colgraph_solve(c, delta)
    assert_same(gpu(cg, c, delta, opts=tiles(cg, **kw)), o, f"{name} {kw}")


def test_tiles_weight_mode(cg):
    rng = np.random.default_rng(7)
    for trial in range(100):
        X, Y, Z = (int(v) for v in rng.integers(1, 8, 3))
        delta = int(rng.integers(0, 4))
        w = rng.integers(-20, 21, size=(X, Y, Z)).astype(np.int32)
        o = oracle.colgraph_solve(w, delta, input_is_weight=True)
        r = gpu(cg, w, delta, weight=True, opts=tiles(cg))
        assert r["flow"] == o["flow"] and np.array_equal(r["mask"], o["mask"]), trial


def test_tiles_rejects_tall_columns(cg):
    c = np.zeros((2, 2, 300), np.int32)
    t = torch.from_numpy(c).cuda()
    h = cg.colgraph_build(t, 1)
    try:
        assert cg.maxflow_solve(h, tiles(cg))[0] == cg.CG_E_INVAL
    finally:
        cg.colgraph_free(h)


@pytest.mark.parametrize("var", [{"CG_RELABEL": "bfs"}, {"CG_RELABEL": "bfs", "CG_BFS_LEVEL_LAUNCHES": "1"},
                                 {"CG_WALK_MIN": "0"}, {"CG_RELABEL": "bfs", "CG_BFS_SMALL": "2048"},
                                 {"CG_RELABEL": "bfs", "CG_BFS_SMALL": "0"}, {"CG_COLGR_SMALL": "0"},
                                 {"CG_COLGR_SMALL": "100000"}, {"CG_GR_SCHEDULE": "1,2,3,5,8,13,21,34"},
                                 {"CG_GR_BETA": "1000"}, {"CG_OPS": "4"},
                                 {"CG_BFS_TRUNC": "64,2"}, {"CG_BFS_TRUNC": "100000000,1"}, {"CG_BFS_TRUNC": "0,0"},
                                 {"CG_BFS_TRUNC": "64,2,0"}, {"CG_BFS_TRUNC": "16,1"}, {"CG_ADAPT_BATCH": "0"},
                                 {"CG_ADAPT_BATCH": "1"}, {"CG_ADAPT_BATCH": "5"},
                                 {"CG_BFS_BU": "1000000,1"}, {"CG_BFS_BU": "2,64"}, {"CG_PRECANCEL": "1"},
                                 {"CG_BFS_DENSE": "1"}, {"CG_BFS_DENSE": "0"}])
def test_schedule_variants(cg, env, var):
    for k, v in var.items():
        env.setenv(k, v)
    for seed in range(1000, 1200):
        c, delta = V.tiny_case(seed)
        assert_same(gpu(cg, c, delta), oracle.colgraph_solve(c, delta), f"{var} seed {seed}")
    for name in ("C1", "C2"):
        c = V.generate(name)
        delta = V.CONFIGS[name].delta
        assert_same(gpu(cg, c, delta), oracle.colgraph_solve(c, delta), f"{var} {name}")


@pytest.mark.parametrize("name", ["C3"])
def test_tiles_full_size(cg, name):
    """C3 on tiles vs the stored oracle result (scripts/make_oracle_golden.py)."""
    import hashlib
    import json
    spec = V.CONFIGS[name]
    c = V.generate(name)
    r = gpu(cg, c, spec.delta, opts=tiles(cg))
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", f"oracle_{name}.json")))
    assert r["flow"] == gold["flow"]
    assert hashlib.sha256(r["surface"].astype("<i4").tobytes()).hexdigest() == gold["surface_sha256"]
    assert hashlib.sha256(r["mask"].tobytes()).hexdigest() == gold["mask_sha256"]
