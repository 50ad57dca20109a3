#!/bin/bash
# profiles/ncu_traffic_c<cfg>.json: DRAM bytes per launch of each modeled
# stage's kernel (one `ncu --set full` capture of the third analyze call).
#   bash scripts/ncu_traffic_run.sh 3    (XS_EVENTS=... to shrink config 3/5)
cfg=${1:-2}
cd "$(dirname "$0")/.."
K='regex:k_bk_sweep|k_bk_hist|k_bk_scatter|k_pass1|k_quantize|k_removal|k_remap'
# 2 warm analyze calls issue 16 launches of these kernels (k_pass1 twice per call)
XS_CONFIG=$cfg XS_CALLS=3 ncu --set full --clock-control none -k "$K" -s 16 -c 8 \
  -o /tmp/r2_traffic_c$cfg python scripts/prof_step.py > /tmp/r2_traffic_c$cfg.log 2>&1
python scripts/ncu_traffic.py /tmp/r2_traffic_c$cfg.ncu-rep > profiles/ncu_traffic_c$cfg.json
cat profiles/ncu_traffic_c$cfg.json
