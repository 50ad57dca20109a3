#!/bin/bash
# A/B of env knobs on the per-stage device times: ab_env.sh "ENV=a ENV2=b" "ENV=c" ...
for v in "$@"; do
  echo "== $v"
  env $v python scripts/stage_times.py 2>&1 | tail -2
done
