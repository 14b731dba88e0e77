"""Host-side logic of the multi-GPU (x-slab) path, exercised with world_size-2 gloo on
CPU: the ncclUniqueId bootstrap, the slab partition of the volume, and reassembly of
per-rank results.  (The device side of the slab algorithm is tested on one GPU by
tests/test_gpu_slabs.py through colgraph_build_slabs.)"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2601_17026_b200 import dist as cgd
    from synth import volumes as V
    nid = cgd.init_nccl_id()
    spec = V.CONFIGS["C1"]
    x0, x1 = cgd.slab(spec.X, rank, world)
    mine = V.generate("C1", x_range=(x0, x1))
    vol = cgd.gather_slabs(mine)
    # per-rank slices of the oracle surface reassemble to the full surface
    full = oracle.colgraph_solve(V.generate("C1"), spec.delta, want_mask=False)["surface"]
    surf = cgd.gather_slabs(full[x0:x1])
    ids = [None] * world
    dist.all_gather_object(ids, nid)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), vol=vol, surf=surf, full=full, x0=x0, x1=x1,
             same_id=all(i == ids[0] for i in ids), idlen=len(nid))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slab_plumbing(tmp_path, world):
    import torch.multiprocessing as mp
    from synth import volumes as V
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    full_vol = V.generate("C1")
    ranges = []
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        assert bool(d["same_id"]) and int(d["idlen"]) == 128
        assert np.array_equal(d["vol"], full_vol)          # slabs tile the volume in rank order
        assert np.array_equal(d["surf"], d["full"])        # per-rank results reassemble
        ranges.append((int(d["x0"]), int(d["x1"])))
    assert ranges[0][0] == 0 and ranges[-1][1] == full_vol.shape[0]
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
