"""The x-slab algorithm's own cost on ONE GPU: the in-process transport runs all slabs on the
same device (so no speedup is possible); the time over the single-slab solve is the overhead
of partitioning (per-sweep halos, label-correcting relabels, top halos).  Diagnostics."""
import json
import os
import statistics
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
    for ns in (1, 2, 4, 8):
        ts, r = [], None
        for rep in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = cg.solve(c, spec.delta, want_mask=False, nslabs=ns)
            torch.cuda.synchronize()
            if rep:
                ts.append((time.perf_counter() - t) * 1000)
        s = r["stats"]
        print(json.dumps({"config": name, "slabs": ns, "flow": r["flow"], "ms": round(statistics.median(ts), 1),
                          "sweeps": s["sweeps"], "global_relabels": s["global_relabels"],
                          "relabel_passes": s["gr_passes"], "ms_gr": round(s["ms_global_relabel"], 1),
                          "ms_sweep": round(s["ms_sweep_kernels"], 1)}), flush=True)
