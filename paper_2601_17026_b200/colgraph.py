"""Thin ctypes binding of libcolgraph.so (include/colgraph.h).  Argument
marshalling only: every step of the path runs in the library's CUDA kernels.
There is no CPU fallback -- importing this module on a box without the built
library raises.

Names follow the C ABI: colgraph_build, maxflow_solve, mincut_extract_surface,
colgraph_free, colgraph_solve_host, colgraph_export_state, cg_slab_range.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CG_LIB") or os.path.join(_PKG, "libcolgraph.so")

STATUS = {0: "CG_OK", 1: "CG_E_INVAL", 2: "CG_E_OVERFLOW", 3: "CG_E_NOMEM", 4: "CG_E_CUDA", 5: "CG_E_NCCL",
          6: "CG_E_EMPTY_COLUMN", 7: "CG_E_STATE", 8: "CG_E_NOT_CONVERGED"}
CG_OK, CG_E_INVAL, CG_E_OVERFLOW, CG_E_EMPTY_COLUMN, CG_E_STATE, CG_E_NOT_CONVERGED = 0, 1, 2, 6, 7, 8


class ColgraphError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: {STATUS.get(status, status)}")
        self.status = status


class cg_dims(ctypes.Structure):
    """delta: Delta_x; delta_y: Delta_y (-1 = isotropic).  Python callers may pass delta as an
    int or as a (delta_x, delta_y) pair."""
    _fields_ = [("X", ctypes.c_int32), ("Y", ctypes.c_int32), ("Z", ctypes.c_int32), ("delta", ctypes.c_int32),
                ("delta_y", ctypes.c_int32)]

    def __init__(self, X=0, Y=0, Z=0, delta=0, delta_y=None):
        if isinstance(delta, (tuple, list)):
            delta, delta_y = delta
        super().__init__(int(X), int(Y), int(Z), int(delta), -1 if delta_y is None else int(delta_y))


class cg_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("nccl_id", ctypes.c_void_p),
                ("device", ctypes.c_int32), ("stream", ctypes.c_void_p)]


class cg_solve_opts(ctypes.Structure):
    _fields_ = [("gr_factor", ctypes.c_float), ("gap_every", ctypes.c_int32), ("check_every", ctypes.c_int32),
                ("max_sweeps", ctypes.c_int64), ("ops_per_sweep", ctypes.c_int32), ("walk_len", ctypes.c_int32),
                ("sweep_kind", ctypes.c_int32), ("tile_steps", ctypes.c_int32), ("tile_relabel_every", ctypes.c_int32)]


class cg_solve_stats(ctypes.Structure):
    _fields_ = [("sweeps", ctypes.c_int64), ("global_relabels", ctypes.c_int64), ("gr_passes", ctypes.c_int64),
                ("work", ctypes.c_int64), ("gap_runs", ctypes.c_int64), ("gap_lifted", ctypes.c_int64),
                ("extract_passes", ctypes.c_int64), ("ms_build", ctypes.c_double), ("ms_solve", ctypes.c_double),
                ("ms_extract", ctypes.c_double), ("ms_global_relabel", ctypes.c_double),
                ("ms_sweeps", ctypes.c_double), ("bytes_per_sweep_alg", ctypes.c_double),
                ("source_capacity", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("ms_sweep_kernels", ctypes.c_double), ("sweep_bytes_alg", ctypes.c_double),
                ("tile_visits", ctypes.c_int64), ("relabel_ops", ctypes.c_int64), ("gr_truncated", ctypes.c_int64),
                ("bk_stages", ctypes.c_int64), ("bk_growths", ctypes.c_int64), ("bk_augmentations", ctypes.c_int64),
                ("bk_orphans", ctypes.c_int64), ("bk_freed", ctypes.c_int64), ("ms_bk_last_stages", ctypes.c_double),
                ("src_terminated", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class cg_bk_opts(ctypes.Structure):
    _fields_ = [("seg_x", ctypes.c_int32), ("seg_y", ctypes.c_int32), ("time_limit_ms", ctypes.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built: run python -m paper_2601_17026_b200.build "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    lib.colgraph_build.restype = ctypes.c_int
    lib.colgraph_build.argtypes = [P(cg_dims), ctypes.c_void_p, ctypes.c_int32, P(cg_dist), P(ctypes.c_void_p)]
    lib.colgraph_build_soft.restype = ctypes.c_int
    lib.colgraph_build_soft.argtypes = [P(cg_dims), ctypes.c_void_p, ctypes.c_int32, P(ctypes.c_int32), ctypes.c_int32,
                                        P(cg_dist), P(ctypes.c_void_p)]
    lib.colgraph_build_slabs_soft.restype = ctypes.c_int
    lib.colgraph_build_slabs_soft.argtypes = [P(cg_dims), ctypes.c_void_p, ctypes.c_int32, P(ctypes.c_int32),
                                              ctypes.c_int32, ctypes.c_int32, P(cg_dist), P(ctypes.c_void_p)]
    lib.colgraph_build_slabs.restype = ctypes.c_int
    lib.colgraph_build_slabs.argtypes = [P(cg_dims), ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, P(cg_dist),
                                         P(ctypes.c_void_p)]
    lib.cg_nccl_unique_id.restype = ctypes.c_int
    lib.cg_nccl_unique_id.argtypes = [ctypes.c_void_p]
    lib.colgraph_build_general.restype = ctypes.c_int
    lib.colgraph_build_general.argtypes = [P(cg_dims), ctypes.c_void_p, ctypes.c_int32, P(ctypes.c_int32),
                                           ctypes.c_void_p, P(ctypes.c_int32), ctypes.c_int32, ctypes.c_int32,
                                           P(cg_dist), P(ctypes.c_void_p)]
    lib.cg_nccl_loopback.restype = ctypes.c_int
    lib.cg_nccl_loopback.argtypes = [ctypes.c_int32]
    lib.maxflow_solve.restype = ctypes.c_int
    lib.maxflow_solve.argtypes = [ctypes.c_void_p, P(cg_solve_opts), P(ctypes.c_int64), P(cg_solve_stats)]
    lib.maxflow_solve_bk.restype = ctypes.c_int
    lib.maxflow_solve_bk.argtypes = [ctypes.c_void_p, P(cg_bk_opts), P(ctypes.c_int64), P(cg_solve_stats)]
    lib.mincut_extract_surface.restype = ctypes.c_int
    lib.mincut_extract_surface.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    lib.colgraph_solve_host.restype = ctypes.c_int
    lib.colgraph_solve_host.argtypes = [P(cg_dims), ctypes.c_void_p, ctypes.c_int32, P(cg_dist), P(cg_solve_opts),
                                        P(ctypes.c_int64), ctypes.c_void_p, ctypes.c_void_p, P(cg_solve_stats)]
    lib.maxflow_export_flow.restype = ctypes.c_int
    lib.maxflow_export_flow.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, P(cg_solve_opts),
                                        ctypes.c_void_p]
    lib.colgraph_export_state.restype = ctypes.c_int
    lib.colgraph_export_state.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    lib.colgraph_stats.restype = ctypes.c_int
    lib.colgraph_stats.argtypes = [ctypes.c_void_p, P(cg_solve_stats)]
    lib.colgraph_free.restype = None
    lib.colgraph_free.argtypes = [ctypes.c_void_p]
    lib.cg_status_str.restype = ctypes.c_char_p
    lib.cg_status_str.argtypes = [ctypes.c_int]
    lib.cg_slab_range.restype = ctypes.c_int
    lib.cg_slab_range.argtypes = [P(cg_dims), ctypes.c_int32, ctypes.c_int32, P(ctypes.c_int32), P(ctypes.c_int32)]
    lib.cg_version.restype = ctypes.c_char_p
    lib.cg_version.argtypes = []
    return lib


_lib = _load()

EXPORTED = ["colgraph_build", "colgraph_build_slabs", "colgraph_build_soft", "colgraph_build_slabs_soft", "colgraph_build_general", "cg_nccl_unique_id", "cg_nccl_loopback", "maxflow_solve", "maxflow_solve_bk", "mincut_extract_surface",
            "maxflow_export_flow", "colgraph_solve_host",
            "colgraph_export_state", "colgraph_stats", "colgraph_free", "cg_status_str", "cg_slab_range", "cg_version"]


def lib():
    return _lib


def version() -> str:
    return _lib.cg_version().decode()


SWEEP_AUTO, SWEEP_TILES, SWEEP_VERTEX = 0, 1, 2


def make_opts(gr_factor=1.0, gap_every=0, check_every=8, max_sweeps=1 << 30, ops_per_sweep=1,
              walk_len=0, sweep_kind=SWEEP_AUTO, tile_steps=0, tile_relabel_every=0) -> cg_solve_opts:
    return cg_solve_opts(float(gr_factor), int(gap_every), int(check_every), int(max_sweeps), int(ops_per_sweep),
                         int(walk_len), int(sweep_kind), int(tile_steps), int(tile_relabel_every))


def _dist(device=0, stream=None, rank=0, nranks=1, nccl_id=None) -> cg_dist:
    return cg_dist(rank, nranks, nccl_id, device, stream)


def _check_dev_int32(t, name):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.int32 and t.is_contiguous()):
        raise TypeError(f"{name} must be a contiguous CUDA int32 tensor")


def colgraph_build_soft(cost, delta, penalty, input_is_weight: bool = False, stream=None, rank=0, nranks=1,
                        nccl_id=None, dims=None):
    """NEXT-1: soft smoothness, penalty = [f(1), ..., f(K)] convex (include/colgraph.h).  With
    nranks > 1: this rank's slab of the full volume dims (as colgraph_build)."""
    _check_dev_int32(cost, "cost")
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(cost.device)
    if dims is None:
        X, Y, Z = cost.shape
        dims = cg_dims(X, Y, Z, delta)
    pen = (ctypes.c_int32 * len(penalty))(*[int(v) for v in penalty])
    h = ctypes.c_void_p()
    idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
    st = _lib.colgraph_build_soft(ctypes.byref(dims), ctypes.c_void_p(cost.data_ptr()), int(bool(input_is_weight)),
                                  pen, len(penalty),
                                  ctypes.byref(_dist(cost.device.index, ctypes.c_void_p(stream.cuda_stream), rank,
                                                     nranks, ctypes.cast(idbuf, ctypes.c_void_p)
                                                     if idbuf is not None else None)), ctypes.byref(h))
    if st != CG_OK:
        raise ColgraphError(st, "colgraph_build_soft")
    return h


def colgraph_build_slabs_soft(cost, delta, penalty, nslabs: int, input_is_weight: bool = False, stream=None):
    """In-process x-slabs of a soft-smoothness graph (include/colgraph.h)."""
    _check_dev_int32(cost, "cost")
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(cost.device)
    X, Y, Z = cost.shape
    dims = cg_dims(X, Y, Z, delta)
    pen = (ctypes.c_int32 * len(penalty))(*[int(v) for v in penalty])
    h = ctypes.c_void_p()
    st = _lib.colgraph_build_slabs_soft(ctypes.byref(dims), ctypes.c_void_p(cost.data_ptr()),
                                        int(bool(input_is_weight)), pen, len(penalty), int(nslabs),
                                        ctypes.byref(_dist(cost.device.index, ctypes.c_void_p(stream.cuda_stream))),
                                        ctypes.byref(h))
    if st != CG_OK:
        raise ColgraphError(st, "colgraph_build_slabs_soft")
    return h


def colgraph_build(cost, delta: int, input_is_weight: bool = False, stream=None, rank=0, nranks=1, nccl_id=None,
                   dims=None):
    """cost: CUDA int32 tensor [X_r, Y, Z] (this rank's slab; dims = full-volume cg_dims when
    nranks > 1, nccl_id = the 128 bytes from nccl_unique_id() shared by all ranks).
    Returns an opaque handle."""
    _check_dev_int32(cost, "cost")
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(cost.device)
    if dims is None:
        X, Y, Z = cost.shape
        dims = cg_dims(X, Y, Z, delta)
    h = ctypes.c_void_p()
    idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
    st = _lib.colgraph_build(ctypes.byref(dims), ctypes.c_void_p(cost.data_ptr()), int(bool(input_is_weight)),
                             ctypes.byref(_dist(cost.device.index, ctypes.c_void_p(stream.cuda_stream), rank, nranks,
                                                ctypes.cast(idbuf, ctypes.c_void_p) if idbuf is not None else None)),
                             ctypes.byref(h))
    if st != CG_OK:
        raise ColgraphError(st, "colgraph_build")
    return h


def deltas4(delta):
    """Edge intervals toward (+x, -x, +y, -y) from an int, (delta_x, delta_y) or a 4-tuple."""
    if isinstance(delta, (tuple, list)):
        if len(delta) == 4:
            return tuple(int(d) for d in delta)
        dx, dy = int(delta[0]), int(delta[1])
        dy = dx if dy == -1 else dy
        return (dx, dx, dy, dy)
    return (int(delta),) * 4


def colgraph_build_general(cost, delta, band=None, penalty=None, nslabs: int = 0, input_is_weight: bool = False,
                           stream=None, rank=0, nranks=1, nccl_id=None, dims=None):
    """NEXT-3 (include/colgraph.h colgraph_build_general): delta int / (dx, dy) / (d+x, d-x, d+y, d-y);
    band: CUDA int32 tensor [X_r, Y, 2] (lo, hi) per column or None; penalty: soft smoothness or None;
    nslabs >= 1: in-process x-slabs; else one slab per process (nranks > 1: NCCL)."""
    _check_dev_int32(cost, "cost")
    if band is not None:
        _check_dev_int32(band, "band")
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(cost.device)
    d4 = deltas4(delta)
    if dims is None:
        X, Y, Z = cost.shape
        dims = cg_dims(X, Y, Z, d4[0], d4[2])
    dl = (ctypes.c_int32 * 4)(*d4)
    pen = (ctypes.c_int32 * len(penalty))(*[int(v) for v in penalty]) if penalty is not None else None
    h = ctypes.c_void_p()
    idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
    st = _lib.colgraph_build_general(ctypes.byref(dims), ctypes.c_void_p(cost.data_ptr()), int(bool(input_is_weight)),
                                     dl, ctypes.c_void_p(band.data_ptr()) if band is not None else None,
                                     pen, len(penalty) if penalty is not None else 0, int(nslabs),
                                     ctypes.byref(_dist(cost.device.index, ctypes.c_void_p(stream.cuda_stream), rank,
                                                        nranks, ctypes.cast(idbuf, ctypes.c_void_p)
                                                        if idbuf is not None else None)), ctypes.byref(h))
    if st != CG_OK:
        raise ColgraphError(st, "colgraph_build_general")
    return h


def colgraph_build_slabs(cost, delta: int, nslabs: int, input_is_weight: bool = False, stream=None):
    """Whole volume `cost` (CUDA int32 [X, Y, Z]) cut into `nslabs` x-slabs inside this process,
    exchanging the same halo messages as NCCL ranks (device-to-device copies)."""
    _check_dev_int32(cost, "cost")
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(cost.device)
    X, Y, Z = cost.shape
    dims = cg_dims(X, Y, Z, delta)
    h = ctypes.c_void_p()
    st = _lib.colgraph_build_slabs(ctypes.byref(dims), ctypes.c_void_p(cost.data_ptr()), int(bool(input_is_weight)),
                                   int(nslabs), ctypes.byref(_dist(cost.device.index,
                                                                   ctypes.c_void_p(stream.cuda_stream))),
                                   ctypes.byref(h))
    if st != CG_OK:
        raise ColgraphError(st, "colgraph_build_slabs")
    return h


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for multi-GPU colgraph_build (rank 0 creates, all ranks share)."""
    buf = ctypes.create_string_buffer(128)
    st = _lib.cg_nccl_unique_id(buf)
    if st != CG_OK:
        raise ColgraphError(st, "cg_nccl_unique_id")
    return buf.raw


def nccl_loopback(enable: bool) -> None:
    """TEST HOOK: route every later NCCL call of this process through the in-process loopback
    transport (all ranks as host threads on one device; include/colgraph.h cg_nccl_loopback)."""
    st = _lib.cg_nccl_loopback(int(bool(enable)))
    if st != CG_OK:
        raise ColgraphError(st, "cg_nccl_loopback")


def maxflow_solve(handle, opts: cg_solve_opts | None = None):
    """Returns (status, |f|, stats dict)."""
    flow = ctypes.c_int64(0)
    stats = cg_solve_stats()
    st = _lib.maxflow_solve(handle, ctypes.byref(opts) if opts is not None else None, ctypes.byref(flow),
                            ctypes.byref(stats))
    return st, int(flow.value), stats.as_dict()


def maxflow_solve_bk(handle, seg_x: int = 0, seg_y: int = 0, time_limit_ms: int = 0):
    """NEXT-4: parallel BK with hierarchical merging (include/colgraph.h).  Returns (status, |f|, stats)."""
    flow = ctypes.c_int64(0)
    stats = cg_solve_stats()
    o = cg_bk_opts(int(seg_x), int(seg_y), int(time_limit_ms))
    st = _lib.maxflow_solve_bk(handle, ctypes.byref(o), ctypes.byref(flow), ctypes.byref(stats))
    return st, int(flow.value), stats.as_dict()


def mincut_extract_surface(handle, surface, mask=None) -> int:
    _check_dev_int32(surface, "surface")
    return _lib.mincut_extract_surface(handle, ctypes.c_void_p(surface.data_ptr()),
                                       ctypes.c_void_p(mask.data_ptr()) if mask is not None else None)


def colgraph_export_state(handle, out) -> int:
    _check_dev_int32(out, "out")
    return _lib.colgraph_export_state(handle, ctypes.c_void_p(out.data_ptr()))


def colgraph_stats(handle) -> dict:
    stats = cg_solve_stats()
    st = _lib.colgraph_stats(handle, ctypes.byref(stats))
    if st != CG_OK:
        raise ColgraphError(st, "colgraph_stats")
    return stats.as_dict()


def maxflow_export_flow(handle, cost, input_is_weight: bool = False, flow=None, opts: cg_solve_opts | None = None,
                        soft_k: int = 0):
    """Phase 2 + flow export (include/colgraph.h).  cost: the CUDA int32 input given to
    colgraph_build.  Returns (status, flow) with flow a CUDA int32 tensor [7 + 4 K, X, Y, Z]:
    s->v, v->t, down, lateral +x, -x, +y, -y, then the soft arcs (soft_k = K for soft graphs)."""
    import torch
    _check_dev_int32(cost, "cost")
    if flow is None:
        flow = torch.empty((7 + 4 * soft_k,) + tuple(cost.shape), dtype=torch.int32, device=cost.device)
    _check_dev_int32(flow, "flow")
    st = _lib.maxflow_export_flow(handle, ctypes.c_void_p(cost.data_ptr()), int(bool(input_is_weight)),
                                  ctypes.byref(opts) if opts is not None else None, ctypes.c_void_p(flow.data_ptr()))
    return st, flow


def colgraph_free(handle) -> None:
    _lib.colgraph_free(handle)


def colgraph_solve_host(cost: np.ndarray, delta: int, input_is_weight: bool = False, want_mask: bool = False,
                        opts: cg_solve_opts | None = None, device: int = 0, stream=None):
    """End-to-end on host buffers (H2D, build, solve, extract, D2H inside the library)."""
    cost = np.ascontiguousarray(cost, dtype=np.int32)
    X, Y, Z = cost.shape
    dims = cg_dims(X, Y, Z, delta)
    surface = np.empty((X, Y), np.int32)
    mask = np.empty((X, Y, Z), np.uint8) if want_mask else None
    flow = ctypes.c_int64(0)
    stats = cg_solve_stats()
    st = _lib.colgraph_solve_host(ctypes.byref(dims), cost.ctypes.data, int(bool(input_is_weight)),
                                  ctypes.byref(_dist(device, stream)), ctypes.byref(opts) if opts is not None else None,
                                  ctypes.byref(flow), surface.ctypes.data, mask.ctypes.data if want_mask else None,
                                  ctypes.byref(stats))
    return {"status": st, "flow": int(flow.value), "surface": surface, "mask": mask, "stats": stats.as_dict()}


def colgraph_solve_host_ptr(cost_host, delta: int, surface_host, mask_host=None, input_is_weight: bool = False,
                            opts: cg_solve_opts | None = None, stream=None):
    """colgraph_solve_host on (pinned) host torch tensors, without extra host copies."""
    X, Y, Z = cost_host.shape
    dims = cg_dims(X, Y, Z, delta)
    flow = ctypes.c_int64(0)
    stats = cg_solve_stats()
    sh = ctypes.c_void_p(stream.cuda_stream) if stream is not None else None
    st = _lib.colgraph_solve_host(ctypes.byref(dims), ctypes.c_void_p(cost_host.data_ptr()),
                                  int(bool(input_is_weight)), ctypes.byref(_dist(0 if stream is None else
                                                                                 stream.device.index, sh)),
                                  ctypes.byref(opts) if opts is not None else None, ctypes.byref(flow),
                                  ctypes.c_void_p(surface_host.data_ptr()),
                                  ctypes.c_void_p(mask_host.data_ptr()) if mask_host is not None else None,
                                  ctypes.byref(stats))
    return {"status": st, "flow": int(flow.value), "stats": stats.as_dict()}


def cg_slab_range(X: int, Y: int, Z: int, delta: int, rank: int, nranks: int):
    dims = cg_dims(X, Y, Z, delta)
    x0, x1 = ctypes.c_int32(), ctypes.c_int32()
    st = _lib.cg_slab_range(ctypes.byref(dims), rank, nranks, ctypes.byref(x0), ctypes.byref(x1))
    if st != CG_OK:
        raise ColgraphError(st, "cg_slab_range")
    return x0.value, x1.value


def solve(cost, delta: int, input_is_weight: bool = False, want_mask: bool = True, opts=None, nslabs: int = 1,
          penalty=None, band=None, bk=None):
    """Device-resident convenience: build -> solve -> extract on a CUDA int32 tensor
    (nslabs > 1: the in-process x-slab path; bk = (seg_x, seg_y) or True: maxflow_solve_bk, NEXT-4).
    Returns dict(status, extract_status, flow, surface (tensor), mask (tensor), stats)."""
    import torch
    X, Y, Z = cost.shape
    if band is not None or (isinstance(delta, (tuple, list)) and len(delta) == 4):
        h = colgraph_build_general(cost, delta, band, penalty, nslabs if nslabs > 1 else 0, input_is_weight)
    elif penalty is not None:
        h = colgraph_build_soft(cost, delta, penalty, input_is_weight) if nslabs == 1 else \
            colgraph_build_slabs_soft(cost, delta, penalty, nslabs, input_is_weight)
    else:
        h = colgraph_build(cost, delta, input_is_weight) if nslabs == 1 else \
            colgraph_build_slabs(cost, delta, nslabs, input_is_weight)
    try:
        if bk is not None and bk is not False:
            sx, sy = (0, 0) if bk is True else bk
            st, flow, stats = maxflow_solve_bk(h, sx, sy)
        else:
            st, flow, stats = maxflow_solve(h, opts)
        surface = torch.empty((X, Y), dtype=torch.int32, device=cost.device)
        mask = torch.empty((X, Y, Z), dtype=torch.uint8, device=cost.device) if want_mask else None
        est = mincut_extract_surface(h, surface, mask) if st == CG_OK else CG_E_STATE
        stats = colgraph_stats(h)
    finally:
        colgraph_free(h)
    return {"status": st, "extract_status": est, "flow": flow, "surface": surface, "mask": mask, "stats": stats}
