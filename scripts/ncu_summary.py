"""Markdown table from an ncu --set full capture (a .ncu-rep, or its
`--page raw --csv` export): per kernel launch, duration, DRAM bytes, achieved
DRAM GB/s and its share of the measured peak, SM throughput, occupancy.

    python scripts/ncu_summary.py gpurun_out/full_c2.ncu-rep "config 2 (1M events)" >> profiles/r01_ncu_summary.md
"""
import csv
import io
import json
import os
import subprocess
import sys

src, title = sys.argv[1], sys.argv[2]
if src.endswith(".ncu-rep"):
    text = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
else:
    text = open(src).read()
rows = list(csv.reader(io.StringIO(text)))
h, units = rows[0], rows[1]
ix = {n: i for i, n in enumerate(h)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(root, "MEASURED_PEAKS.json")) else 6650.0


def val(r, name):
    return float(r[ix[name]].replace(",", "")) * scale.get(units[ix[name]], 1.0)


print(f"\n### {title}\n")
print("| kernel | time (us) | DRAM read+write (MB) | DRAM GB/s | % of peak | SM throughput % | warps active % | regs |")
print("|---|---|---|---|---|---|---|---|")
for r in rows[2:]:
    name = r[ix["Kernel Name"]].replace("void ", "").split("(")[0].replace("xs::", "")[:40]
    t = val(r, "gpu__time_duration.sum")
    b = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    gbs = b / t / 1e9 if t else 0.0
    print(f"| {name} | {t * 1e6:.1f} | {b / 1e6:.1f} | {gbs:.0f} | {100 * gbs / peak:.1f} | "
          f"{float(r[ix['sm__throughput.avg.pct_of_peak_sustained_elapsed']]):.1f} | "
          f"{float(r[ix['sm__warps_active.avg.pct_of_peak_sustained_active']]):.1f} | "
          f"{r[ix['launch__registers_per_thread']]} |")
