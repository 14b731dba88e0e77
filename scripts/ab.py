"""A/B timing of solver variants (diagnostics): median wall time of build+solve+extract over
reps, per config.  Variants are env settings applied in subprocesses.
usage: python scripts/ab.py C3,C4,C5 reps 'NAME:ENV=V,ENV=V' ...   (AB_OPTS={json} -> cg_solve_opts fields;
pass it inside a variant as AB_OPTS={"gap_every":1} -- no commas inside: use ; between fields)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, os, sys, time, statistics
sys.path.insert(0, ROOT)
import torch
from paper_2601_17026_b200 import colgraph as cg
from synth import volumes as V
reps = int(sys.argv[2])
for name in sys.argv[1].split(","):
    spec = V.CONFIGS[name]
    c = torch.from_numpy(V.generate(name)).cuda()
    ts, r = [], None
    for rep in range(reps + 1):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = cg.solve(c, spec.delta, want_mask=False, opts=cg.make_opts(**json.loads(os.environ.get("AB_OPTS", "{}"))))
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        if rep:
            ts.append(dt * 1000)
            st = r["stats"]
            print(json.dumps({"rep": rep, "ms": round(dt * 1000, 1), "sweeps": st["sweeps"], "grs": st["global_relabels"],
                              "ms_gr": round(st["ms_global_relabel"], 1), "ms_sw": round(st["ms_sweep_kernels"], 1),
                              "ms_solve": round(st["ms_solve"], 1), "ms_build": round(st["ms_build"], 1),
                              "ms_extract": round(st["ms_extract"], 1)}), file=sys.stderr, flush=True)
    s = r["stats"]
    print(json.dumps({"config": name, "flow": r["flow"], "med_ms": round(statistics.median(ts), 1), "all": [round(t) for t in ts],
                      "min_ms": round(min(ts), 1), "sweeps": s["sweeps"], "grs": s["global_relabels"],
                      "ms_gr": round(s["ms_global_relabel"], 1), "ms_sw": round(s["ms_sweep_kernels"], 1),
                      "ns_per_op": round(1e6 * s["ms_sweep_kernels"] / max(1, s["work"]), 3)}), flush=True)
'''.replace("ROOT", repr(ROOT))

cfgs, reps = sys.argv[1], sys.argv[2]
for var in sys.argv[3:]:
    name, _, envs = var.partition(":")
    env = dict(os.environ)
    for kv in filter(None, envs.split(",")):
        k, _, v = kv.partition("=")
        env[k] = v.replace(";", ",")
    out = subprocess.run([sys.executable, "-c", CHILD, cfgs, reps], env=env, capture_output=True, text=True,
                         timeout=600)
    for line in out.stdout.splitlines():
        d = json.loads(line)
        print(f"{name:12s} {d['config']} flow={d['flow']} med={d['med_ms']} all={d['all']} sweeps={d['sweeps']} "
              f"grs={d['grs']} gr_ms={d['ms_gr']} sw_ms={d['ms_sw']} ns/op={d['ns_per_op']}", flush=True)
    if out.returncode:
        print(name, "FAILED", out.stderr[-2000:])
    elif os.environ.get("AB_VERBOSE"):
        print(out.stderr)
