"""Time the NEXT-4 solver (maxflow_solve_bk, parallel BK with hierarchical merging) beside the
push-relabel path on the same configs; one JSON line per (config, segment size).

    python scripts/bk_timing.py C2,C3 4x4,8x8 [time_limit_ms]
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_17026_b200 import colgraph as cg  # noqa: E402
from synth import volumes as V  # noqa: E402


def one(name, c, delta, seg, limit):
    t = torch.from_numpy(c).cuda()
    torch.cuda.synchronize()
    h = cg.colgraph_build(t, delta)
    try:
        t0 = time.perf_counter()
        if seg is None:
            st, flow, stats = cg.maxflow_solve(h)
        else:
            st, flow, stats = cg.maxflow_solve_bk(h, seg[0], seg[1], limit)
        surf = torch.empty(c.shape[:2], dtype=torch.int32, device="cuda")
        est = cg.mincut_extract_surface(h, surf) if st == 0 else -1
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
    finally:
        cg.colgraph_free(h)
    gold = os.path.join(ROOT, "tests", "golden", f"oracle_{name}.json")
    gflow = json.load(open(gold))["flow"] if os.path.exists(gold) else None
    keys = ("bk_stages", "bk_growths", "bk_augmentations", "bk_orphans", "bk_freed", "ms_bk_last_stages", "sweeps",
            "global_relabels")
    return {"config": name, "solver": "bk" if seg else "push-relabel", "seg": seg, "status": st, "extract_status": est,
            "flow": flow, "flow_matches_golden": (flow == gflow) if gflow is not None else None,
            "ms_solve_extract": round(ms, 2), **{k: stats[k] for k in keys}}


def main():
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2"]
    segs = [tuple(int(v) for v in s.split("x")) for s in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["4x4"])]
    limit = int(sys.argv[3]) if len(sys.argv) > 3 else 120000
    for name in names:
        spec = V.CONFIGS[name]
        c = V.generate(name)
        one(name, c, spec.delta, None, limit)  # warm-up
        print(json.dumps(one(name, c, spec.delta, None, limit)), flush=True)
        for seg in segs:
            print(json.dumps(one(name, c, spec.delta, seg, limit)), flush=True)


if __name__ == "__main__":
    main()
