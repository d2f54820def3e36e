#!/usr/bin/env bash
# Build the UNMODIFIED reference (graphann, /root/reference/pkg) into oracle/_ref/.
#
# Test/bench infrastructure only: the result is the CPU checker and the CPU
# baseline arm of bench.py, never the product path.  The reference sources are
# copied to a scratch dir under /tmp (the mount is read-only), its own Cython
# module `_core.pyx` is compiled with the reference's own flags (-O3, see
# pkg/setup.py:19-30) and the built package is installed as `graphann_ref`
# under oracle/_ref/ (git-ignored, but shipped to the GPU box by gpurun).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${GGNN_REFERENCE:-/root/reference}/pkg"
OUT="$HERE/_ref"
if [ ! -d "$SRC" ]; then
  echo "reference not present at $SRC; keeping existing $OUT" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/ggnn_ref_build.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
chmod -R u+w "$TMP/pkg"
( cd "$TMP/pkg" && python setup.py -q build_ext --inplace >/dev/null 2>"$TMP/build.log" ) || { cat "$TMP/build.log" >&2; exit 1; }
rm -rf "$OUT/graphann_ref"
mkdir -p "$OUT"
cp -r "$TMP/pkg/src/graphann" "$OUT/graphann_ref"
# the package imports itself relatively, so renaming the directory is enough
rm -f "$OUT/graphann_ref/_core.c"
python - "$OUT" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import graphann_ref
assert graphann_ref.backend.BACKEND == "compiled", graphann_ref.backend.BACKEND
print("built reference:", graphann_ref.__file__, graphann_ref.backend.BACKEND)
PY
