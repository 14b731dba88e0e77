"""One build+solve+extract of a config (for ncu launch lists / captures)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2601_17026_b200 import colgraph as cg  # noqa: E402
from synth import volumes as V  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
spec = V.CONFIGS[name]
c = torch.from_numpy(V.generate(name)).cuda()
r = cg.solve(c, spec.delta, want_mask=False)
torch.cuda.synchronize()
import json  # noqa: E402
print(json.dumps({"config": name, "status": r["status"], "flow": r["flow"],
                  **{k: r["stats"][k] for k in ("sweeps", "global_relabels", "gr_passes", "kernel_launches",
                                                 "sweep_bytes_alg", "ms_sweep_kernels") if k in r["stats"]}}))
