"""Summarise an ncu --set full report: key metrics and the SASS instructions with the most warp-stall
samples (the source page), for a quick hot-spot read.

    python tools/ncu_hot.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = ["Duration", "Issue Slots Busy", "Achieved Occupancy", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "Registers Per Thread", "Block Limit Registers", "Memory Throughput",
        "DRAM Throughput", "L2 Hit Rate"]
for r in csv.reader(io.StringIO(det)):
    if len(r) > 14 and r[12] in want:  # [..., section, metric name, unit, value]
        print(f"  {r[12]}: {r[14]} {r[13]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = [i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r]
if not h:
    sys.exit(0)
hdr = rows[h[0]]
iw, isrc, iad = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Address")
data = []
for r in rows[h[0] + 1:]:
    try:
        data.append((float(r[iw] or 0), r[iad], r[isrc]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1.0
print(f"  stall samples: {tot:.0f}")
for v, a, s in sorted(data, key=lambda d: -d[0])[:top]:
    print(f"  {v / tot * 100:5.1f}%  {a[-5:]}  {s.strip()[:90]}")
