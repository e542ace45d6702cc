"""Aggregate an ncu --csv launch list per kernel name: launches, total / average device time,
share of the listed time and, when the list carries dram__bytes_read.sum / dram__bytes_write.sum,
the DRAM bytes per launch and the achieved HBM GB/s (against the measured 6.55 TB/s copy rate of
MEASURED_PEAKS.json).  ncu's per-launch times are cold-cache and serialised: compare shares.

    python tools/summarize_launches.py launches.csv
"""
import csv
import sys
from collections import defaultdict

HBM_GBS = 6550.0
path = sys.argv[1]
rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
idi = hdr.index("ID") if "ID" in hdr else None
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
per = defaultdict(dict)  # launch id -> metric -> value (bytes / ns)
name_of = {}
for n, r in enumerate(rows[1:]):
    lid = r[idi] if idi is not None else n
    v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    per[lid][r[mi]] = v
    name_of[lid] = r[ki].split("(")[0]
tot, cnt, rd, wr = defaultdict(float), defaultdict(int), defaultdict(float), defaultdict(float)
for lid, m in per.items():
    nm = name_of[lid]
    tot[nm] += m.get("gpu__time_duration.sum", 0.0)
    cnt[nm] += 1
    rd[nm] += m.get("dram__bytes_read.sum", 0.0)
    wr[nm] += m.get("dram__bytes_write.sum", 0.0)
T = sum(tot.values())
print(f"{'kernel':52s} {'launches':>8s} {'total_us':>11s} {'avg_us':>8s} {'share':>6s} {'MB/launch':>10s} {'GB/s':>8s} {'frac_hbm':>8s}")
for nm, v in sorted(tot.items(), key=lambda x: -x[1]):
    b = (rd[nm] + wr[nm]) / cnt[nm]
    gbs = (rd[nm] + wr[nm]) / v if v > 0 else 0.0  # bytes / ns = GB/s
    print(f"{nm[:52]:52s} {cnt[nm]:8d} {v / 1e3:11.1f} {v / cnt[nm] / 1e3:8.2f} {v / T:6.3f} {b / 1e6:10.3f} {gbs:8.1f} "
          f"{gbs / HBM_GBS:8.3f}")
print(f"{'TOTAL':52s} {sum(cnt.values()):8d} {T / 1e3:11.1f}")
