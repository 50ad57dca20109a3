"""Key metrics of kernels in an ncu report: `python scripts/ncu_brief.py REP [KERNEL_REGEX]`."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
args = ["ncu", "-i", rep, "--page", "details", "--csv"]
if len(sys.argv) > 2:
    args += ["-k", "regex:" + sys.argv[2]]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.DictReader(io.StringIO(out)))
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Executed Ipc Active", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "Grid Size"]
seen = {}
for r in rows:
    key = (r["ID"], r["Kernel Name"].split("(")[0])
    if r["Metric Name"] in want:
        seen.setdefault(key, {})[r["Metric Name"]] = f"{r['Metric Value']} {r['Metric Unit']}".strip()
for (i, name), m in seen.items():
    print(f"[{i}] {name}")
    print("   " + "; ".join(f"{k}={m[k]}" for k in want if k in m))
