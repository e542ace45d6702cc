"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel name."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    v = float(r[vi].replace(",", ""))
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':60s} {'launches':>9s} {'total_us':>12s} {'avg_us':>9s} {'share':>7s}")
for name, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{name[:60]:60s} {cnt[name]:9d} {v/1e3:12.1f} {v/cnt[name]/1e3:9.2f} {v/T:7.3f}")
print(f"{'TOTAL':60s} {sum(cnt.values()):9d} {T/1e3:12.1f}")
