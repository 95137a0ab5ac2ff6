#!/usr/bin/env bash
# Build a scratch copy of the reference package (read-only at /root/reference)
# with its Cython extension, so make_golden.py can import it.  Only used in the
# build container to (re)generate tests/golden/*.npz; nothing on the GPU box
# reads /root/reference.
set -euo pipefail
DEST=${1:-/tmp/refbuild}
if [ ! -f "$DEST/src/rtcur/_backend/_core.c" ] || ! ls "$DEST"/src/rtcur/_backend/_core*.so >/dev/null 2>&1; then
  rm -rf "$DEST"
  cp -r /root/reference/pkg "$DEST"
  (cd "$DEST" && python setup.py build_ext --inplace >/dev/null)
fi
echo "$DEST/src"
