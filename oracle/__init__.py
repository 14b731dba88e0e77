"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct explicit-graph max-flow / min-cut (Dinitz and
Edmonds-Karp, §2) for Wu-Chen column graphs (PAPER.md:42-43
§1.2, Eqs. 2-7 §1.3).  See oracle.c's header for every formula and citation.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  The product library
(paper_2601_17026_b200) never imports, links or executes it, and this
package imports nothing from the product.

Parity status per function:
  colgraph_solve  -- pinned (brute-force surfaces, 1-D DP, closed forms,
                     worked examples, invariants, metamorphic relations)
  graph_maxflow   -- pinned (brute-force minimum cuts on small graphs,
                     SPEC.md hand examples)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

STATUS = {0: "OK", 1: "INVAL", 3: "NOMEM", 6: "EMPTY_COLUMN"}
CHECK_BITS = {
    "capacity": 1 << 0,
    "antisymmetry": 1 << 1,
    "conservation": 1 << 2,
    "value": 1 << 3,
    "t_not_in_S": 1 << 4,
    "cut_eq_flow": 1 << 5,
}
ALL_CHECKS = sum(CHECK_BITS.values())
ALGOS = {"dinic": 0, "ek": 1, "pr": 2}


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-shared", "-fPIC", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i32p = ctypes.POINTER(ctypes.c_int32)
        i64p = ctypes.POINTER(ctypes.c_int64)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        lib.oracle_colgraph_solve.restype = ctypes.c_int
        lib.oracle_colgraph_solve.argtypes = [i32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_int, ctypes.c_int, i64p, i32p, u8p, i32p, i64p]
        lib.oracle_colgraph_solve_soft.restype = ctypes.c_int
        lib.oracle_colgraph_solve_soft.argtypes = [i32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                   ctypes.c_int, i32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, i64p,
                                                   i32p, u8p, i32p, i64p]
        lib.oracle_colgraph_solve_general.restype = ctypes.c_int
        lib.oracle_colgraph_solve_general.argtypes = [i32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, i32p, i32p,
                                                      i32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, i64p, i32p, u8p,
                                                      i32p, i64p]
        lib.oracle_graph_maxflow.restype = ctypes.c_int
        lib.oracle_graph_maxflow.argtypes = [ctypes.c_int, ctypes.c_int, i32p, i32p, i64p, ctypes.c_int,
                                             ctypes.c_int, ctypes.c_int, i64p, u8p, i32p]
        lib.oracle_graph_check.restype = ctypes.c_int
        lib.oracle_graph_check.argtypes = [ctypes.c_int, ctypes.c_int, i32p, i32p, i64p, i64p, i64p, ctypes.c_int,
                                           ctypes.c_int, u8p, ctypes.c_int64, i32p]
        _lib = lib
    return _lib


def _ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def deltas4(delta):
    """Edge intervals toward (+x, -x, +y, -y): delta is an int (isotropic), (delta_x, delta_y)
    (anisotropic, NEXT-3) or a 4-tuple (general proper-ordered interval: the pair p, q = p + x
    satisfies S(q) - S(p) in [-delta[0], delta[1]], likewise y with delta[2], delta[3])."""
    if isinstance(delta, (tuple, list)):
        if len(delta) == 2:
            dx, dy = int(delta[0]), int(delta[1])
            dy = dx if dy == -1 else dy
            return (dx, dx, dy, dy)
        return tuple(int(d) for d in delta)
    return (int(delta),) * 4


def colgraph_solve(c: np.ndarray, delta, input_is_weight: bool = False, algo: str = "dinic",
                   want_mask: bool = True, penalty=None, band=None) -> dict:
    """Solve the column graph of cost (or weight) volume c[X][Y][Z].  delta: see deltas4.
    penalty: optional convex soft-smoothness penalty [f(1), .., f(K)], K >= max(delta) (NEXT-1:
    finite arcs of capacity f(k+1) - 2 f(k) + f(k-1)).  band: optional int32 [X, Y, 2] (lo, hi) per
    column, the narrow band the surface is confined to (NEXT-3; costs only).

    Returns dict(status, flow, surface[X,Y] int32, mask[X,Y,Z] uint8 or None,
    checks (bit set), n_arcs).
    """
    lib = _load()
    c = np.ascontiguousarray(c, dtype=np.int32)
    X, Y, Z = c.shape
    flow = np.zeros(1, np.int64)
    surface = np.zeros((X, Y), np.int32)
    mask = np.zeros((X, Y, Z), np.uint8) if want_mask else None
    checks = np.zeros(1, np.int32)
    n_arcs = np.zeros(1, np.int64)
    dl4 = np.array(deltas4(delta), np.int32)
    pen = np.ascontiguousarray(penalty, dtype=np.int32) if penalty is not None else None
    bnd = np.ascontiguousarray(band, dtype=np.int32).reshape(X * Y * 2) if band is not None else None
    st = lib.oracle_colgraph_solve_general(_ptr(c, ctypes.c_int32), X, Y, Z, _ptr(dl4, ctypes.c_int32),
                                           _ptr(bnd, ctypes.c_int32) if bnd is not None else None,
                                           _ptr(pen, ctypes.c_int32) if pen is not None else None,
                                           len(pen) if pen is not None else 0, int(bool(input_is_weight)),
                                           ALGOS[algo], _ptr(flow, ctypes.c_int64), _ptr(surface, ctypes.c_int32),
                                           _ptr(mask, ctypes.c_uint8) if want_mask else None,
                                           _ptr(checks, ctypes.c_int32), _ptr(n_arcs, ctypes.c_int64))
    return {"status": int(st), "flow": int(flow[0]), "surface": surface, "mask": mask,
            "checks": int(checks[0]), "n_arcs": int(n_arcs[0])}


def graph_maxflow(nn: int, arcs, s: int, t: int, algo: str = "dinic") -> dict:
    """Max flow on an explicit arc list [(u, v, cap), ...] over nodes 0..nn-1."""
    lib = _load()
    arcs = list(arcs)
    tails = np.array([a[0] for a in arcs], np.int32)
    heads = np.array([a[1] for a in arcs], np.int32)
    caps = np.array([a[2] for a in arcs], np.int64)
    flow = np.zeros(1, np.int64)
    side = np.zeros(nn, np.uint8)
    checks = np.zeros(1, np.int32)
    st = lib.oracle_graph_maxflow(nn, len(arcs), _ptr(tails, ctypes.c_int32), _ptr(heads, ctypes.c_int32),
                                  _ptr(caps, ctypes.c_int64), s, t, ALGOS[algo], _ptr(flow, ctypes.c_int64),
                                  _ptr(side, ctypes.c_uint8), _ptr(checks, ctypes.c_int32))
    return {"status": int(st), "flow": int(flow[0]), "source_side": side.astype(bool), "checks": int(checks[0])}


def graph_check(nn: int, arcs, res_fwd, res_rev, s: int, t: int, source_side, flow: int) -> int:
    """check_invariants on a GIVEN residual state: arcs [(u, v, cap)], res_fwd[i] / res_rev[i] the
    residuals of arc i and of its reverse slot, source_side the claimed S, flow the claimed |f|.
    Returns the CHECK_BITS that hold (test entry point that pins the checker itself)."""
    lib = _load()
    arcs = list(arcs)
    tails = np.array([a[0] for a in arcs], np.int32)
    heads = np.array([a[1] for a in arcs], np.int32)
    caps = np.array([a[2] for a in arcs], np.int64)
    rf = np.ascontiguousarray(res_fwd, np.int64)
    rr = np.ascontiguousarray(res_rev, np.int64)
    side = np.ascontiguousarray(source_side, np.uint8)
    checks = np.zeros(1, np.int32)
    st = lib.oracle_graph_check(nn, len(arcs), _ptr(tails, ctypes.c_int32), _ptr(heads, ctypes.c_int32),
                                _ptr(caps, ctypes.c_int64), _ptr(rf, ctypes.c_int64), _ptr(rr, ctypes.c_int64), s, t,
                                _ptr(side, ctypes.c_uint8), int(flow), _ptr(checks, ctypes.c_int32))
    if st != 0:
        raise ValueError(f"oracle_graph_check: status {st}")
    return int(checks[0])
