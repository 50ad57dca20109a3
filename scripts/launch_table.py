"""Summarise an ncu --csv launch list (gpu__time_duration.sum) for the last N
engine calls: per-kernel time, count and share.  Usage:
    python scripts/launch_table.py launches.csv [marker_kernel] [marker_skip]"""
import csv
import sys

path = sys.argv[1]
marker = sys.argv[2] if len(sys.argv) > 2 else "k_init_stats"
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 2
lines = [ln for ln in open(path) if ln.startswith('"')]
rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
idx = [i for i, r in enumerate(rows) if marker in r["Kernel Name"]]
last = rows[idx[-skip]:] if len(idx) >= skip else rows
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = {}
tot = 0.0
for r in last:
    name = r["Kernel Name"]
    name = name.split("(")[0].replace("void ", "")[:80]
    v = float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
    tot += v
    a = agg.setdefault(name, [0.0, 0])
    a[0] += v
    a[1] += 1
print(f"launches {len(last)}  total {tot:.1f} us")
for name, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{v:8.1f} us {100 * v / tot:5.1f}% {c:3d}x  {name}")
