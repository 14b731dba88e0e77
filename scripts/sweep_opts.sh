#!/bin/bash
# usage: scripts/sweep_opts.sh CONFIGS 'ENV1' 'ENV2' ...   (each ENV is a set of VAR=val for one run)
cfgs=$1; shift
for e in "$@"; do
  echo "== $e"
  env $e timeout 300 python scripts/diag_solve.py $cfgs 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(d['config'], d['status'], d['flow'], 'wall_ms', d['wall_ms'], 'sweeps', d['sweeps'], 'GR', d['global_relabels'], 'levels', d['gr_passes'], 'ms_gr', d['ms_global_relabel'], 'ms_sw', d['ms_sweep_kernels'], 'work', d['work'])
"
done
