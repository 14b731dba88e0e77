"""The NCCL x-slab path itself (colgraph_build with nranks > 1), executed on ONE GPU.

cg_nccl_loopback(1) (include/colgraph.h, csrc/nccl_loopback.h) swaps libnccl for an in-process
transport; every rank is a host thread with its own stream and its own slab, and the library runs
its NCCL code unchanged: the communicator cache (comm_acquire), grouped ncclSend/ncclRecv halos
(transfer), ncclAllReduce counters (gsum).  This is the paper's column segmentation with a boundary
exchange and per-level synchronisation (§3.2.1-3.2.2).  Results must be
bit-identical to the oracle (unique by SURVEY.md §8(c) c3)."""
import json
import os
import threading

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
    colgraph.nccl_loopback(True)
    yield colgraph
    colgraph.nccl_loopback(False)


def solve_ranks(cg, c, delta, R, penalty=None, weight=False, opts=None, want_mask=True, flow_export=False):
    """One host thread per rank (ctypes releases the GIL), each with its own stream and slab."""
    c = np.ascontiguousarray(c, np.int32)
    X, Y, Z = c.shape
    nid = cg.nccl_unique_id()
    dims = cg.cg_dims(X, Y, Z, delta)
    slabs, streams = [], []
    for r in range(R):
        x0, x1 = cg.cg_slab_range(X, Y, Z, 0, r, R)
        slabs.append(torch.from_numpy(c[x0:x1].copy()).cuda())
        streams.append(torch.cuda.Stream())
    torch.cuda.synchronize()
    out = [None] * R
    err = [None] * R

    def rank_main(r):
        try:
            s = streams[r]
            if penalty is None:
                h = cg.colgraph_build(slabs[r], delta, weight, stream=s, rank=r, nranks=R, nccl_id=nid, dims=dims)
            else:
                h = cg.colgraph_build_soft(slabs[r], delta, penalty, weight, stream=s, rank=r, nranks=R, nccl_id=nid,
                                           dims=dims)
            try:
                st, flow, _ = cg.maxflow_solve(h, opts)
                xr = slabs[r].shape[0]
                with torch.cuda.stream(s):
                    surf = torch.empty((xr, Y), dtype=torch.int32, device="cuda")
                    mask = torch.empty((xr, Y, Z), dtype=torch.uint8, device="cuda") if want_mask else None
                est = cg.mincut_extract_surface(h, surf, mask) if st == 0 else -1
                fl = None
                if flow_export and st == 0:
                    kk = max(delta) if isinstance(delta, (tuple, list)) else delta
                    planes = 7 + (4 * kk if penalty is not None else 0)
                    with torch.cuda.stream(s):
                        fl = torch.empty(planes * xr * Y * Z, dtype=torch.int32, device="cuda")
                    fst, fl = cg.maxflow_export_flow(h, slabs[r], weight, fl, opts)
                    fl = (fst, fl)
                stats = cg.colgraph_stats(h)
            finally:
                cg.colgraph_free(h)
            s.synchronize()
            out[r] = {"status": st, "ext": est, "flow": flow, "surface": surf.cpu().numpy(),
                      "mask": mask.cpu().numpy() if want_mask else None, "stats": stats, "flow_export": fl}
        except Exception as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "a rank hung"
    for e in err:
        if e is not None:
            raise e
    flows = {o["flow"] for o in out}
    assert len(flows) == 1, flows  # |f| is global on every rank
    return {"status": max(o["status"] for o in out), "ext": max(o["ext"] for o in out), "flow": out[0]["flow"],
            "surface": np.concatenate([o["surface"] for o in out], 0),
            "mask": np.concatenate([o["mask"] for o in out], 0) if want_mask else None, "ranks": out}


def same(r, o, ctx, mask=True):
    assert r["status"] == 0 and r["ext"] == 0, (ctx, r["status"], r["ext"])
    assert r["flow"] == o["flow"], (ctx, r["flow"], o["flow"])
    assert np.array_equal(r["surface"], o["surface"]), ctx
    if mask:
        assert np.array_equal(r["mask"], o["mask"]), ctx


def test_random_tiny_ranks(cg):
    rng = np.random.default_rng(11)
    done = 0
    for seed in range(4000, 4120):
        c, delta = V.tiny_case(seed)
        X = c.shape[0]
        if X < 2:
            continue
        R = int(rng.integers(2, min(X, 4) + 1))
        same(solve_ranks(cg, c, delta, R), oracle.colgraph_solve(c, delta), f"seed {seed} {c.shape} d{delta} R{R}")
        done += 1
    assert done > 60


@pytest.mark.parametrize("R", [2, 3, 5])
def test_c1_ranks(cg, R):
    c = V.generate("C1")
    same(solve_ranks(cg, c, 2, R), oracle.colgraph_solve(c, 2), f"C1 R{R}")


@pytest.mark.parametrize("R", [2, 4])
def test_c2_ranks(cg, R):
    c = V.generate("C2")
    r = solve_ranks(cg, c, 3, R)
    same(r, oracle.colgraph_solve(c, 3), f"C2 R{R}")
    # every rank exchanged halos every sweep and agreed on every counter
    for o in r["ranks"]:
        assert o["stats"]["sweeps"] == r["ranks"][0]["stats"]["sweeps"]
        assert o["stats"]["global_relabels"] == r["ranks"][0]["stats"]["global_relabels"]


def test_c3_two_ranks_vs_golden(cg):
    import hashlib
    g = json.load(open(os.path.join(GOLDEN_DIR, "oracle_C3.json")))
    c = V.generate("C3")
    r = solve_ranks(cg, c, 2, 2, want_mask=False)
    assert r["status"] == 0 and r["flow"] == g["flow"]
    assert hashlib.sha256(r["surface"].astype("<i4").tobytes()).hexdigest() == g["surface_sha256"]


def test_weight_mode_ranks(cg):
    rng = np.random.default_rng(3)
    for k in range(30):
        X, Y, Z = int(rng.integers(2, 6)), int(rng.integers(1, 5)), int(rng.integers(1, 7))
        w = rng.integers(-9, 10, size=(X, Y, Z)).astype(np.int32)
        delta = int(rng.integers(0, 3))
        o = oracle.colgraph_solve(w, delta, input_is_weight=True)
        r = solve_ranks(cg, w, delta, int(rng.integers(2, X + 1)), weight=True)
        assert r["flow"] == o["flow"], k
        assert np.array_equal(r["mask"], o["mask"]), k


def test_soft_ranks(cg):
    rng = np.random.default_rng(8)
    for k in range(40):
        X, Y, Z = int(rng.integers(2, 6)), int(rng.integers(1, 5)), int(rng.integers(2, 8))
        c = rng.integers(0, 10, size=(X, Y, Z)).astype(np.int32)
        delta = int(rng.integers(1, 4))
        pen = list(np.cumsum(np.cumsum(rng.integers(0, 4, size=delta))))
        o = oracle.colgraph_solve(c, delta, penalty=pen)
        r = solve_ranks(cg, c, delta, int(rng.integers(2, X + 1)), penalty=pen)
        same(r, o, f"soft {k} {c.shape} d{delta} pen {pen}")


def test_options_ranks(cg):
    """Relabel / check cadence knobs change the collective schedule, never the result."""
    c = V.generate("C1")
    o = oracle.colgraph_solve(c, 2)
    for kw in ({"check_every": 1}, {"check_every": 256}, {"gr_factor": 0.05}, {"walk_len": -1}):
        same(solve_ranks(cg, c, 2, 3, opts=cg.make_opts(**kw)), o, f"C1 {kw}")


def test_flow_export_ranks(cg):
    """Phase 2 + flow export over NCCL ranks: conservation and value per rank slab."""
    c = V.generate("C1")
    X, Y, Z = c.shape
    o = oracle.colgraph_solve(c, 2)
    r = solve_ranks(cg, c, 2, 2, flow_export=True)
    same(r, o, "C1 export")
    for o_r in r["ranks"]:
        fst, fl = o_r["flow_export"]
        assert fst == 0
    # inflow into t summed over ranks = |f|
    into_t = sum(int(o_r["flow_export"][1].view(7, -1)[1].sum()) for o_r in r["ranks"])
    assert into_t == o["flow"]
