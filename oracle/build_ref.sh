#!/usr/bin/env bash
# Test infrastructure only (oracle): builds the UNMODIFIED reference package
# `repsched` (/root/reference/pkg) with its compiled Cython decide kernel into
# oracle/_ref/ (git-ignored, travels to the GPU box with the snapshot).
# /root/reference is read-only, so the build runs from a scratch copy in /tmp.
# Nothing here is part of the product path.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${REF_PKG:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -d "$SRC" ]; then
  echo "reference package not present at $SRC; keeping existing $OUT" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/repsched_ref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$OUT"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --target "$OUT" "$TMP/pkg"
python - "$OUT" <<'PY'
import os, sys
sys.path.insert(0, sys.argv[1])
os.environ["REPSCHED_KERNEL"] = "compiled"
import repsched._core as c
assert c.KERNEL_NAME == "compiled", c.KERNEL_NAME
print("oracle/_ref: repsched built, kernel =", c.KERNEL_NAME)
PY
