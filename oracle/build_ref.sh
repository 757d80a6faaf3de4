#!/usr/bin/env bash
# Build the UNMODIFIED reference package (ilans, incl. its Cython kernel
# pkg/src/ilans/_core.pyx) from /root/reference into oracle/_ref/.
#
# Test infrastructure only: oracle/_ref is the checker and the CPU baseline
# ("cpu_baseline.kind": "reference"), never the product. /root/reference is
# read-only, so the build runs on a scratch copy under /tmp; only the built
# package lands in oracle/_ref/ (git-ignored, but it travels to the GPU box).
set -euo pipefail
here="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
src="${ILANS_REF_SRC:-/root/reference/pkg}"
out="$here/_ref"
if [ ! -d "$src" ]; then
  echo "build_ref: $src not present; keeping existing $out" >&2
  exit 0
fi
tmp="$(mktemp -d /tmp/ilans_ref.XXXXXX)"
trap 'rm -rf "$tmp"' EXIT
cp -r "$src" "$tmp/pkg"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --target "$tmp/site" "$tmp/pkg" >/dev/null
rm -rf "$out"
mkdir -p "$out"
cp -r "$tmp/site/ilans" "$out/ilans"
# the reference's own test suite travels with it (git-ignored like the rest
# of _ref): integration/install_into_reference.py runs it against the B200
# backend on the GPU box, where /root/reference does not exist
cp -r "$src/tests" "$out/tests"
python - "$out" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
from ilans import backend
assert backend.EXT is not None, "reference _core extension did not build"
print("build_ref: ilans", backend.available(), "->", sys.argv[1])
PY
