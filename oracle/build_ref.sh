#!/bin/bash
# Build the reference package (xstrace, Python + its Cython sweep kernel) from
# /root/reference/pkg into oracle/_ref/ (git-ignored, travels to the GPU box).
# The build runs from a scratch copy because setup.py writes into its tree.
# Used only as the bench's `--impl reference` arm and as a golden-vector
# generator; the product never imports it.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC=${1:-/root/reference/pkg}
[ -d "$SRC" ] || { echo "reference not present ($SRC); skipping"; exit 0; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
python -m pip install -q --no-index --no-build-isolation --no-deps --target "$HERE/_ref" "$TMP/pkg"
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$HERE/_ref'); import xstrace.overlap as o; print('reference built, native sweep:', o.HAVE_NATIVE_SWEEP)"
