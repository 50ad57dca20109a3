"""profiles/ncu_traffic.json from an `ncu --set full` report: DRAM bytes
(dram__bytes_read.sum + dram__bytes_write.sum) per launch of each pipeline
stage's kernels, averaged over the captured launches.  bench.py reports it as
roofline.traffic for the dominant stage.

    python scripts/ncu_traffic.py gpurun_out/full_r01b.ncu-rep > profiles/ncu_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

STAGE_KERNELS = {  # stage -> kernels launched once per stage occurrence
    "sweep_scan_hist": ["k_bk_sweep"],
    "endpoint_keygen": ["k_bk_hist"],
    "endpoint_sort": ["k_bk_scatter"],
    "pass1_validate_spans": ["k_pass1"],
    "quantize_scan": ["k_quantize"],
    "removal_scan": ["k_removal"],
    "remap": ["k_remap"],
}

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ix = {n: i for i, n in enumerate(h)}
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def val(r, name):
    u = units[ix[name]]
    return float(r[ix[name]].replace(",", "")) * scale.get(u, 1)


per = {}
for r in rows[2:]:
    name = r[ix["Kernel Name"]]
    b = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    for stage, ks in STAGE_KERNELS.items():
        if any(name.startswith(k) or f"::{k}" in name or name.startswith(f"void {k}") for k in ks):
            per.setdefault(stage, []).append(b)
res = {k: round(sum(v) / len(v)) for k, v in per.items()}
res["_source"] = f"ncu --set full --clock-control none, {rep.split('/')[-1]}: mean DRAM bytes per launch"
print(json.dumps(res, indent=1))
