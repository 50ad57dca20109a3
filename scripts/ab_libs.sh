#!/bin/bash
# A/B of in-tree library variants (paper_2102_04285_b200/lib_<V>.so) on the
# per-stage device times: bash scripts/ab_libs.sh "3 2" "A B"
cd "$(dirname "$0")/.."
for cfg in ${1:-3 2}; do
for v in ${2:-A B} ${2:-A B}; do
  echo "== cfg $cfg lib $v"
  XS_CONFIG=$cfg XS_LIB_PATH=$PWD/paper_2102_04285_b200/lib_$v.so timeout 300 python scripts/stage_times.py 2>&1 | tail -2
done
done
