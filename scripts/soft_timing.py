"""Time the soft-smoothness solve (colgraph_build_soft + maxflow_solve + extract) per config
with a convex penalty; print |f| and the optimality identity (diagnostics)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_17026_b200 import colgraph as cg  # noqa: E402
from synth import volumes as V  # noqa: E402

PEN = [4, 11, 22, 37]
for name in (sys.argv[1] if len(sys.argv) > 1 else "C2,C3,C4").split(","):
    spec = V.CONFIGS[name]
    pen = PEN[:spec.delta]
    c = torch.from_numpy(V.generate(name)).cuda()
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = cg.solve(c, spec.delta, want_mask=False, penalty=pen)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    s = r["stats"]
    # phase 2 + flow export of the soft graph
    h = cg.colgraph_build_soft(c, spec.delta, pen)
    st1, _, _ = cg.maxflow_solve(h, None)
    torch.cuda.synchronize()
    t = time.perf_counter()
    st2, F = cg.maxflow_export_flow(h, c, soft_k=spec.delta)
    torch.cuda.synchronize()
    export_ms = (time.perf_counter() - t) * 1000
    fs = int(F[0].sum(dtype=torch.int64))
    cg.colgraph_free(h)
    del F
    print(json.dumps({"config": name, "penalty": pen, "status": r["status"], "flow": r["flow"],
                      "export_status": st2, "export_ms": round(export_ms, 1), "export_sum_source_flow": fs,
                      "ms": round(dt * 1000, 1), "ms_solve": round(s["ms_solve"], 1), "sweeps": s["sweeps"],
                      "global_relabels": s["global_relabels"], "ms_gr": round(s["ms_global_relabel"], 1),
                      "mnodes_s": round(spec.n / dt / 1e6, 1)}), flush=True)
