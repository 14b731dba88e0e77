"""Copy the evidence of a GPU session (gpurun_out/) into profiles/ under a round/commit tag:
bench lines, per-config solver stats, the ncu launch-list summary, key counters of the
ncu --set full captures, and profiles/traffic.json (the bench's `traffic` field).
usage: python scripts/save_profiles.py TAG"""
import csv
import gzip
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1]
KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__thread_inst_executed_per_inst_executed.ratio"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}


def ncu_summary(rep, name):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    caps = [{k + (f" [{units[hdr.index(k)]}]" if units[hdr.index(k)] else ""): r[hdr.index(k)] for k in KEYS
             if k in hdr} for r in rows[2:]]
    per = []
    for r in rows[2:]:
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(k)
            b += float(r[i]) * SCALE[units[i]]
        per.append(b)
    json.dump({"captures": caps, "dram_bytes_per_launch": per}, open(os.path.join(PROF, f"{tag}_ncu_{name}.json"), "w"),
              indent=1)
    return sum(per) / len(per)


for src, dst in [("bench.log", "bench_c4.json"), ("bench_ref.log", "bench_reference_c4.json"),
                 ("diag.log", "diag_all_configs.jsonl"), ("gpu_tests.log", "gpu_tests.txt")]:
    p = os.path.join(OUT, src)
    if os.path.exists(p):
        shutil.copy(p, os.path.join(PROF, f"{tag}_{dst}"))
if os.path.exists(os.path.join(OUT, "launches.csv")):
    s = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), os.path.join(OUT, "launches.csv")],
                       capture_output=True, text=True).stdout
    open(os.path.join(PROF, f"{tag}_launch_summary_c4.txt"), "w").write(s)
    with open(os.path.join(OUT, "launches.csv"), "rb") as f, gzip.open(os.path.join(PROF, f"{tag}_launches_c4.csv.gz"), "wb") as g:
        g.write(f.read())
for rep, name in [("prof_walk.ncu-rep", "k_walk_ws"), ("prof_bfs.ncu-rep", "k_bfs_run"),
                  ("prof_passes.ncu-rep", "relabel_passes")]:
    p = os.path.join(OUT, rep)
    if os.path.exists(p):
        avg = ncu_summary(p, name)
# the bench's `traffic`: DRAM bytes of EVERY sweep launch of one C4 solve, with that solve's
# own algorithmic bytes (profile_one.py's line in sweep_traffic.log)
st_csv, st_log = os.path.join(OUT, "sweep_traffic.csv"), os.path.join(OUT, "sweep_traffic.log")
if os.path.exists(st_csv) and os.path.exists(st_log):
    import io
    lines = open(st_csv).read().splitlines()
    i0 = next(k for k, l in enumerate(lines) if l.startswith('"ID"'))
    per = {}
    for r in csv.DictReader(io.StringIO("\n".join(lines[i0:]))):
        if r["Metric Name"].startswith("dram__bytes"):
            per[r["ID"]] = per.get(r["ID"], 0.0) + float(r["Metric Value"].replace(",", "")) * SCALE[r["Metric Unit"]]
    alg = next(json.loads(l) for l in open(st_log) if l.startswith("{"))
    tot, n = sum(per.values()), len(per)
    json.dump({"kernel": "k_walk_ws / k_sweep_v (all sweep launches of one C4 solve)",
               "sweep_dram_bytes_per_launch": tot / n,
               "sweep_alg_bytes_per_launch_same_run": alg["sweep_bytes_alg"] / n,
               "traffic_over_alg": tot / alg["sweep_bytes_alg"], "launches": n, "dram_bytes_total": tot,
               "alg_bytes_total": alg["sweep_bytes_alg"],
               "note": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over EVERY k_walk_ws/k_sweep_v launch of "
                       "one C4 solve (scripts/gpu_session.sh); the algorithmic bytes are that same solve's "
                       "(profile_one.py), run with the relabel schedule of an unprofiled solve replayed "
                       "(CG_GR_SCHEDULE) so its sweeps match the bench's.",
               "source": f"profiles/{tag}_sweep_traffic_c4.csv.gz"}, open(os.path.join(PROF, "traffic.json"), "w"),
              indent=1)
    with open(st_csv, "rb") as f, gzip.open(os.path.join(PROF, f"{tag}_sweep_traffic_c4.csv.gz"), "wb") as g:
        g.write(f.read())
print("saved", tag)
