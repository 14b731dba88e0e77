"""Inspect the residual state in the middle of a solve (diagnostics only)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2601_17026_b200 import colgraph as cg  # noqa: E402
from synth import volumes as V  # noqa: E402

name = sys.argv[1]
stops = [int(x) for x in sys.argv[2].split(",")]
spec = V.CONFIGS[name]
c = torch.from_numpy(V.generate(name)).cuda()
n = spec.n
for ms in stops:
    h = cg.colgraph_build(c, spec.delta)
    st, flow, stats = cg.maxflow_solve(h, cg.make_opts(max_sweeps=ms, check_every=16))
    out = torch.empty(8 * n, dtype=torch.int32, device="cuda")
    cg.colgraph_export_state(h, out)
    cg.colgraph_free(h)
    s = out.view(8, spec.X, spec.Y, spec.Z).cpu().numpy()
    E, H, T, D = s[0], s[1], s[2], s[3]
    INF = n + 1
    fin = H < INF
    act = (E > 0) & fin
    Tsum = T.astype(np.int64).sum()
    print(f"--- {name} after {stats['sweeps']} sweeps, GR {stats['global_relabels']}: flow so far {flow}")
    ea = E[act].astype(np.int64)
    print(f" active {act.sum()}  excess on active: sum {ea.sum()} median {np.median(ea) if ea.size else 0} max {ea.max() if ea.size else 0}")
    einf = E[(E > 0) & ~fin].astype(np.int64)
    print(f" stranded (E>0, H=INF) excluding base: {((E>0)&~fin)[:,:,1:].sum()} vertices, excess {E[:,:,1:][((E>0)&~fin)[:,:,1:]].astype(np.int64).sum()}")
    print(f" remaining sink capacity: {Tsum}, T>0 vertices {int((T>0).sum())}, finite-label T>0 {int(((T>0)&fin).sum())}")
    za = act.sum(axis=(0, 1))
    zt = (T > 0).sum(axis=(0, 1))
    print(" active by z-bin(16):", [int(za[z:z+16].sum()) for z in range(0, spec.Z, 16)])
    print(" T>0 by z-bin(16):  ", [int(zt[z:z+16].sum()) for z in range(0, spec.Z, 16)])
    ha = H[act]
    if ha.size:
        print(" active label pctiles 10/50/90/max:", np.percentile(ha, [10, 50, 90]).tolist(), int(ha.max()))
    # columns with active vertices
    cols = act.any(axis=2)
    print(f" columns with active: {cols.sum()} of {spec.X*spec.Y}")
    # spatial clustering: active per column hist
    apc = act.sum(axis=2)[cols]
    print(" active per active column pctiles 50/90/max:", np.percentile(apc, [50, 90]).tolist(), int(apc.max()))
