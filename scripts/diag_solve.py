"""Solve configs on the GPU and print |f|, status and solver statistics (diagnostics only)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2601_17026_b200 import colgraph as cg  # noqa: E402
from synth import volumes as V  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C1", "C2", "C3", "C4", "C5"]
kw = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
for name in names:
    spec = V.CONFIGS[name]
    c = torch.from_numpy(V.generate(name)).cuda()
    runs = []
    for rep in range(4):  # 1 warm-up + 3 timed; report the median run
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = cg.solve(c, spec.delta, want_mask=False, opts=cg.make_opts(**kw))
        torch.cuda.synchronize()
        if rep:
            runs.append((time.perf_counter() - t, r))
    runs.sort(key=lambda p: p[0])
    dt, r = runs[len(runs) // 2]
    s = r["stats"]
    keep = {k: (round(v, 2) if isinstance(v, float) else v) for k, v in s.items()}
    print(json.dumps({"config": name, "status": r["status"], "ext": r["extract_status"], "flow": r["flow"],
                      "wall_ms": round(dt * 1000, 1), "mnodes_s": round(spec.n / dt / 1e6, 1), **keep}), flush=True)
