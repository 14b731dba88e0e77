"""Height statistics after the initial global relabel and after the solve (diagnostics)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2601_17026_b200 import colgraph as cg  # noqa: E402
from synth import volumes as V  # noqa: E402

for name in sys.argv[1].split(","):
    spec = V.CONFIGS[name]
    c = torch.from_numpy(V.generate(name)).cuda()
    n = spec.n
    for label, ms in (("initial", 0), ("final", 1 << 30)):
        h = cg.colgraph_build(c, spec.delta)
        st, flow, stats = cg.maxflow_solve(h, cg.make_opts(max_sweeps=ms))
        out = torch.empty(8 * n, dtype=torch.int32, device="cuda")
        cg.colgraph_export_state(h, out)
        cg.colgraph_free(h)
        s = out.view(8, spec.X, spec.Y, spec.Z)
        E, H, T, D = s[0], s[1], s[2], s[3]
        INF = n + 1
        fin = H < INF
        hf = H[fin].float()
        act = (E > 0) & fin
        print(f"{name} {label}: status={st} finite={fin.float().mean().item():.3f} maxH={int(H[fin].max()) if fin.any() else -1} "
              f"meanH={hf.mean().item():.1f} p99H={hf.quantile(0.99).item() if hf.numel() < 16_000_000 else -1:.0f} "
              f"active={int(act.sum())} E>0={int((E>0).sum())} T>0={int((T>0).sum())} D>0={int((D>0).sum())} "
              f"Lpos={int((s[4:]>0).sum())}", flush=True)
        zs = torch.arange(spec.Z, device="cuda")
        fz = fin.float().mean(dim=(0, 1))
        print("   finite fraction by z (every Z/16):", [round(float(fz[z]), 2) for z in range(0, spec.Z, max(1, spec.Z // 16))])
        az = act.float().sum(dim=(0, 1))
        print("   active by z (every Z/16):", [int(az[z]) for z in range(0, spec.Z, max(1, spec.Z // 16))])
        if fin.any():
            hist = torch.bincount(H[fin].long().clamp(max=4095))
            print("   H histogram (first 40):", hist[:40].tolist(), " count>=4095:", int(hist[4095:].sum()) if hist.numel() > 4095 else 0)
