#!/bin/sh
# Build recipe for oracle/_ref/: the reference package itself (`polyprec`,
# pure Python over numpy/scipy), installed unmodified from /root/reference
# so that bench.py's reference arm and CPU baseline can run the reference's
# own code path on the GPU box (where /root/reference does not exist).
# Output only into oracle/_ref/ (git-ignored, not gpurun-ignored).  The
# build copies the source tree to a temporary directory first because
# /root/reference is read-only.  Run from the repo root (build() does).
set -e
SRC=/root/reference/pkg
OUT="$(cd "$(dirname "$0")" && pwd)/_ref"
[ -d "$SRC" ] || { echo "build_ref: $SRC absent (GPU box): using the prebuilt $OUT"; exit 0; }
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$OUT"
python -m pip install --quiet --no-index --no-deps --no-build-isolation --target "$OUT" "$TMP/pkg"
python -c "import sys; sys.path.insert(0, '$OUT'); import polyprec; print('build_ref: polyprec', polyprec.__version__, 'in', '$OUT')"
