"""Regenerate BASELINE.md's "Measured results" section from profiles/<tag>_*.
usage: python scripts/make_baseline_table.py <tag>   (e.g. r01_late_7b92e68)"""
import json, sys
T = sys.argv[1]
H = T.rsplit('_', 1)[-1]
diag = [json.loads(l) for l in open(f'profiles/{T}_diag_all_configs.jsonl')]
bench = json.loads(open(f'profiles/{T}_bench_c4.json').read().strip().splitlines()[-1])
ref = json.loads(open(f'profiles/{T}_bench_reference_c4.json').read().strip().splitlines()[-1])
tr = json.load(open('profiles/traffic.json'))
wk = json.load(open(f'profiles/{T}_ncu_k_walk.json'))['captures']
ra = bench['roofline_random_access']
n = {'C1': 8192, 'C2': 2097152, 'C3': 16777216, 'C4': 67108864, 'C5': 100663296}
rows = []
for d in diag:
    t = (d['ms_build'] + d['ms_solve'] + d['ms_extract']) / 1000
    rows.append(f"| {d['config']} | 1 | {t:.4f} | {n[d['config']] / t / 1e6:.1f} | {d['sweeps']} | {d['global_relabels']} | "
                f"{d['ms_global_relabel']:.1f} / {d['ms_sweep_kernels']:.1f} | exact |")
rf = bench['roofline']
mm = bench.get('ms_per_step_min_median_max', [bench['ms_per_step']] * 3)
table = f"""## Measured results (round 1, one B200, commit {H})

Library time (build + solve + extract from the library's own timers; the median of 3 runs
after a warm-up, `scripts/diag_solve.py`).  Parity: |f|, minimal source set and surface bit-identical to the
CPU oracle -- C1, C2 and the tiny sweeps live, C3/C4 against stored oracle results, C5
through |f| = cost(surface) + K0 with a Delta-feasible surface (its stored oracle result is
still being computed on the CPU).

| Config | GPUs | time-to-min-cut (s) | Mnodes/s | sweeps | global relabels | relabel / sweep ms | parity |
|---|---|---|---|---|---|---|---|
{chr(10).join(rows)}

Headline (`bench.py`, C4, 5 timed steps, CUDA events, SM clock {bench['clocks']['sm_mhz']:.0f} MHz, no
throttle reasons): **{bench['ms_per_step']:.1f} ms per step = {bench['value']:.1f} Mnodes/s** (per-step min /
median / max {mm[0]:.1f} / {mm[1]:.1f} / {mm[2]:.1f} ms: the lock-free schedule occasionally needs one more
global relabel); through the
host API with the 256 MiB H2D copy and the surface D2H inside the timed region:
{bench['e2e']['value']:.1f} Mnodes/s.  The CPU oracle (single-threaded Dinic) runs at
{bench['cpu_baseline']['value']:.3f} Mnodes/s on a crop of the same volume (`--impl reference`: {ref['value']:.3f} Mnodes/s).

Roofline of the dominant kernel (push-relabel sweep, `k_walk` / `k_sweep_v`): algorithmic
{rf['achieved']:.0f} GB/s = **{100 * rf['frac']:.1f} % of the measured 6,457 GB/s copy peak** (44 B per
push/relabel operation).  ncu (`profiles/{T}_ncu_k_walk.json`, early launches):
{float(wk[0]['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed [%]']):.0f} % of DRAM peak, L2 hit
{float(wk[0]['lts__t_sector_hit_rate.pct [%]']):.0f} %, {float(wk[0]['smsp__thread_inst_executed_per_inst_executed.ratio']):.1f} active threads per warp
instruction -- a divergent, scattered traversal whose DRAM traffic over every sweep launch of
a solve is {tr['traffic_over_alg']:.1f}x its algorithmic bytes (`profiles/traffic.json`).  Its access-pattern
bound is the B200's random 32-byte record gather rate, measured at 625-750 GB/s (12 % of the
copy peak, `profiles/r01_random_gather.json`): against it the sweep runs at
{100 * ra['frac']:.0f} %.  The >= 40 %
per-sweep target of BASELINE.json (a streaming figure) is not met; DESIGN.md §6 explains
why and lists every measured alternative.

Multi-GPU (x-slabs over NCCL): implemented and verified bit-exact through the in-process
slab transport on one GPU; not measured on 2/4/8 GPUs in round 1 (one GPU available).
"""
s = open('BASELINE.md').read()
a = s.index('## Measured results')
b = s.index('## CPU baseline plan')
open('BASELINE.md', 'w').write(s[:a] + table + '\n' + s[b:])
print(table)
