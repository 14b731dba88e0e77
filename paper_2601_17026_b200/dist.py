"""Multi-GPU plumbing for the x-slab path (one process per GPU, torch.distributed for
bootstrap only; every step of the solve runs in libcolgraph.so over NCCL).

  init_nccl_id()      rank 0 asks the library for an ncclUniqueId, broadcast to all ranks
  slab(X, r, R)       this rank's x-range (cg_slab_range: larger slabs first)
  gather_slabs(a)     reassemble per-rank slab arrays along x (results / tests)
  solve_slab(...)     colgraph_build(nranks=R) -> maxflow_solve -> mincut_extract_surface
"""
from __future__ import annotations

import numpy as np

from . import colgraph as cg


def _dist():
    import torch.distributed as dist
    if not dist.is_initialized():
        raise RuntimeError("torch.distributed is not initialised")
    return dist


def init_nccl_id() -> bytes:
    """128-byte ncclUniqueId, identical on every rank (created by rank 0)."""
    import torch
    dist = _dist()
    cuda = dist.get_backend() == "nccl"
    buf = torch.zeros(128, dtype=torch.uint8)
    if dist.get_rank() == 0:
        buf.copy_(torch.frombuffer(bytearray(cg.nccl_unique_id()), dtype=torch.uint8))
    if cuda:
        buf = buf.cuda()
    dist.broadcast(buf, 0)
    return bytes(buf.cpu().numpy().tobytes())


def slab(X: int, rank: int, nranks: int) -> tuple[int, int]:
    return cg.cg_slab_range(X, 1, 1, 0, rank, nranks)


def gather_slabs(local: np.ndarray) -> np.ndarray:
    """Concatenate every rank's slab array along axis 0 (ranks in order) on every rank."""
    dist = _dist()
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, np.ascontiguousarray(local))
    return np.concatenate(parts, axis=0)


def solve_slab(cost_slab, dims: tuple, rank: int, nranks: int, nccl_id: bytes, opts=None, stream=None,
               want_mask: bool = False):
    """Collective solve of this rank's slab (CUDA int32 [X_r, Y, Z]) of the full volume dims=(X, Y, Z, delta).
    Returns dict(status, extract_status, flow (global), surface (slab tensor), mask, stats)."""
    import torch
    X, Y, Z, delta = dims
    d = cg.cg_dims(X, Y, Z, delta)
    h = cg.colgraph_build(cost_slab, delta, rank=rank, nranks=nranks, nccl_id=nccl_id, dims=d, stream=stream)
    try:
        st, flow, _ = cg.maxflow_solve(h, opts)
        xr = cost_slab.shape[0]
        surface = torch.empty((xr, Y), dtype=torch.int32, device=cost_slab.device)
        mask = torch.empty((xr, Y, Z), dtype=torch.uint8, device=cost_slab.device) if want_mask else None
        est = cg.mincut_extract_surface(h, surface, mask) if st == cg.CG_OK else cg.CG_E_STATE
        stats = cg.colgraph_stats(h)
    finally:
        cg.colgraph_free(h)
    return {"status": st, "extract_status": est, "flow": flow, "surface": surface, "mask": mask, "stats": stats}
