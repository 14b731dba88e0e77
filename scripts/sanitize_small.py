"""Small cases through every kernel family (for compute-sanitizer runs): vertex walks,
single-hop sweeps, persistent BFS, level BFS, x-slabs, tiles, phase 2, anisotropy."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_17026_b200 import colgraph as cg  # noqa: E402
from synth import volumes as V  # noqa: E402

cases = [(V.generate("C1"), 2), (V.tiny(5, 7, 5, 40, 255), (1, 3)), (V.tiny(6, 3, 9, 70, 9), 0)]
for c, d in cases:
    t = torch.from_numpy(np.ascontiguousarray(c)).cuda()
    for opts in (None, cg.make_opts(walk_len=-1), cg.make_opts(sweep_kind=cg.SWEEP_TILES)):
        r = cg.solve(t, d, opts=opts)
        assert r["status"] == 0, r["status"]
    r = cg.solve(t, d, nslabs=min(3, c.shape[0]))
    assert r["status"] == 0
    h = cg.colgraph_build(t, d)
    cg.maxflow_solve(h, None)
    st, F = cg.maxflow_export_flow(h, t)
    assert st == 0
    cg.colgraph_free(h)
torch.cuda.synchronize()
print("sanitize cases ok")
