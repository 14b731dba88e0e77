"""Summarise an ncu --csv launch list: time share per kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("cg::", "")
    tot[name] += float(r[vi].replace(",", ""))
    cnt[name] += 1
unit = "ns"
allt = sum(tot.values())
print(f"total {allt/1e6:.3f} ms over {sum(cnt.values())} launches")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:28s} launches={cnt[k]:7d} total={tot[k]/1e6:9.3f} ms share={tot[k]/allt*100:5.1f}% avg={tot[k]/cnt[k]/1e3:8.2f} us")
