#!/usr/bin/env bash
# Build the REAL reference package (rtcur: pure Python + its one Cython
# extension rtcur._backend._core) into oracle/_ref/ -- test/baseline
# infrastructure, never imported by the product.
#
# The sources are compiled where they lie under /root/reference (via a
# throw-away copy in /tmp, because the build writes generated C next to the
# .pyx and /root/reference is read-only); only the installed package lands in
# oracle/_ref/ (git-ignored, but it travels to the GPU box with the snapshot).
# Users: bench.py --impl reference (the timed CPU reference arm) and the
# cpu_baseline leg of bench.py.  Needs Cython + setuptools + numpy (present in
# this image); no network (pip --no-index).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -d "$SRC" ]; then
  echo "reference sources not found at $SRC" >&2
  exit 1
fi
if ls "$OUT"/rtcur/_backend/_core*.so >/dev/null 2>&1; then
  exit 0
fi
TMP="$(mktemp -d /tmp/rtcur_ref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$OUT"
python -m pip install -q --no-index --no-build-isolation --no-deps --target "$OUT" "$TMP/pkg"
ls "$OUT"/rtcur/_backend/_core*.so >/dev/null
