"""Write tests/golden/oracle_<C>.json (flow, surface/mask sha256) for full-size configs.

Calls only oracle/ and synth/ (never the CUDA path).
Usage: python scripts/make_oracle_golden.py C3 [C4 ...]   (ORACLE_ALGO=pr|dinic|ek, default dinic)
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from synth import volumes as V  # noqa: E402

for name in sys.argv[1:]:
    spec = V.CONFIGS[name]
    c = V.generate(name)
    sha = V.sha256_volume(c)
    assert sha == V.MANIFEST[name]
    t = time.time()
    algo = os.environ.get("ORACLE_ALGO", "dinic")
    r = oracle.colgraph_solve(c, spec.delta, want_mask=True, algo=algo)
    dt = time.time() - t
    assert r["status"] == 0 and r["checks"] == oracle.ALL_CHECKS, (r["status"], r["checks"])
    out = {"config": name, "input_sha256": sha, "delta": spec.delta, "flow": r["flow"],
           "surface_sha256": hashlib.sha256(r["surface"].astype("<i4").tobytes()).hexdigest(),
           "mask_sha256": hashlib.sha256(r["mask"].tobytes()).hexdigest(),
           "surface_min": int(r["surface"].min()), "surface_max": int(r["surface"].max()),
           "n_explicit_arcs": r["n_arcs"], "oracle_seconds": round(dt, 1), "oracle_algo": algo,
           "checks": "capacity, antisymmetry, conservation, value, t not in S, cut == flow",
           "written_by": "scripts/make_oracle_golden.py (oracle/ + synth/ only)"}
    with open(os.path.join(ROOT, "tests", "golden", f"oracle_{name}.json"), "w") as f:
        json.dump(out, f, indent=1)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", f"oracle_{name}_surface.npz"), surface=r["surface"])
    print(name, out, flush=True)
