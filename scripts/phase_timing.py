"""Per-call wall times of build / solve / extract / free over reps (diagnostics)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2601_17026_b200 import colgraph as cg  # noqa: E402
from synth import volumes as V  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
spec = V.CONFIGS[name]
c = torch.from_numpy(V.generate(name)).cuda()
surf = torch.empty((spec.X, spec.Y), dtype=torch.int32, device="cuda")
for rep in range(reps):
    t = [time.perf_counter()]
    torch.cuda.synchronize()
    h = cg.colgraph_build(c, spec.delta)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    st, flow, stats = cg.maxflow_solve(h, None)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    cg.mincut_extract_surface(h, surf)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    cg.colgraph_free(h)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    d = [round((b - a) * 1000, 1) for a, b in zip(t, t[1:])]
    print(json.dumps({"rep": rep, "build": d[0], "solve": d[1], "extract": d[2], "free": d[3],
                      "lib_ms_solve": round(stats["ms_solve"], 1)}), flush=True)
