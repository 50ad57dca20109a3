#!/bin/bash
# Build libxstrace_b200.so for sm_100a (B200).  Cross-compiles without a GPU.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
OUT="${XS_OUT:-$HERE/../libxstrace_b200.so}"
OBJ="${XS_OBJ:-$HERE/../../build/obj}"
mkdir -p "$OBJ"
NVCC=${NVCC:-nvcc}
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wno-deprecated-declarations -Wno-deprecated-declarations --expt-relaxed-constexpr -I$HERE/../../include ${XS_NVCC_EXTRA:-}"
pids=()
for f in "$HERE"/*.cu; do
  b=$(basename "$f" .cu)
  $NVCC $FLAGS -c "$f" -o "$OBJ/$b.o" &
  pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT" "$OBJ"/*.o -lcudart
echo "built $OUT"
