"""Top SASS lines by warp-stall samples from `ncu -i X --page source --csv --print-source sass -k K`."""
import csv
import sys

rows = list(csv.reader(sys.stdin))
h = rows[0]
ix = {n: i for i, n in enumerate(h)}
key = "Warp Stall Sampling (All Samples)"
data = []
for r in rows[1:]:
    if len(r) != len(h):
        continue
    try:
        data.append((float(r[ix[key]] or 0), r[ix["Address"]], r[ix["Source"]].strip()))
    except ValueError:
        continue
tot = sum(d[0] for d in data) or 1
top = int(sys.argv[1]) if len(sys.argv) > 1 else 30
for v, a, src in sorted(data, reverse=True)[:top]:
    print(f"{100 * v / tot:5.1f}% {a[-5:]} {src}")
