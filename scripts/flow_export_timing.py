"""Time phase 2 + flow export (maxflow_export_flow) after a solve, per config (diagnostics;
the flow checks themselves are in tests/test_gpu_flow.py)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2601_17026_b200 import colgraph as cg  # noqa: E402
from synth import volumes as V  # noqa: E402

for name in (sys.argv[1] if len(sys.argv) > 1 else "C3,C4").split(","):
    spec = V.CONFIGS[name]
    c = torch.from_numpy(V.generate(name)).cuda()
    F = torch.empty((7, spec.X, spec.Y, spec.Z), dtype=torch.int32, device="cuda")
    for rep in range(3):
        h = cg.colgraph_build(c, spec.delta)
        st, flow, s1 = cg.maxflow_solve(h, None)
        torch.cuda.synchronize()
        t = time.perf_counter()
        st2, _ = cg.maxflow_export_flow(h, c, flow=F)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) * 1000
        s2 = cg.colgraph_stats(h)
        cg.colgraph_free(h)
    fs = int(F[0].sum(dtype=torch.int64)); ft = int(F[1].sum(dtype=torch.int64))
    print(json.dumps({"config": name, "status": st2, "flow": flow, "sum_source_flow": fs, "sum_sink_flow": ft,
                      "phase2_ms": round(dt, 1), "phase1_ms": round(s1["ms_solve"], 1),
                      "phase2_sweeps": s2["sweeps"] - s1["sweeps"],
                      "phase2_relabels": s2["global_relabels"] - s1["global_relabels"]}), flush=True)
