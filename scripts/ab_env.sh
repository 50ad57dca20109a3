#!/bin/bash
# A/B timing of the analyse step under environment variants (GPU box).
# usage: scripts/ab_env.sh "VAR=a" "VAR=b" ...
for v in "$@"; do
  echo "== $v"
  env $v python scripts/step_timeline.py 2>/dev/null | grep analyze
done
