"""Per-phase (barrier-separated) instruction and stall breakdown of one kernel
from an ncu report: `python scripts/ncu_phases.py REP KERNEL_REGEX UNITS`
(UNITS = the work items the kernel processed, e.g. keys, for per-unit counts).
Also prints the top stall reasons per phase."""
import csv
import io
import subprocess
import sys

rep, kre, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre,
                      "-c", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
# a report holding several kernels repeats the header (and a kernel-name
# line) before each: keep the first kernel's rows only
cut = next((i for i, r in enumerate(rows[1:], 1) if r and (r[0] == "Address" or r[0] == "Kernel Name")), len(rows))
rows = rows[:cut]
ix = {n: i for i, n in enumerate(h)}
stalls = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
tot_s = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in rows[1:] if len(r) == len(h))
tot_i = 0
seg = None


def new_seg():
    return {"i": 0.0, "s": 0, "st": {k: 0 for k in stalls}, "n": 0}


seg = new_seg()
segs = []
for r in rows[1:]:
    if len(r) != len(h):
        continue
    ie = int(r[ix["Instructions Executed"]] or 0)
    tot_i += ie
    seg["i"] += ie * 32 / units
    seg["s"] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    for k in stalls:
        seg["st"][k] += int(r[ix[k]] or 0)
    seg["n"] += 1
    src = r[ix["Source"]]
    if "BAR.SYNC" in src or "EXIT" in src:
        seg["end"] = src.strip()[:40]
        segs.append(seg)
        seg = new_seg()
print(f"total thread-instr/unit {tot_i * 32 / units:.1f}  stall samples {tot_s}")
for g in segs:
    if g["i"] < 1 and g["s"] < tot_s * 0.01:
        continue
    top = sorted(g["st"].items(), key=lambda x: -x[1])[:3]
    print(f"{g['n']:5d} sass  {g['i']:7.1f}/unit  stall {100 * g['s'] / tot_s:5.1f}%  "
          + " ".join(f"{k[6:]}={100 * v / tot_s:.1f}" for k, v in top) + f"  | {g.get('end', '')}")
