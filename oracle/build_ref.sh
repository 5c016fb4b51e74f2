#!/usr/bin/env bash
# Builds the UNMODIFIED reference package (color-rl 0.1.0, /root/reference/pkg)
# with its Cython kernel backend into oracle/_ref/ (git-ignored build output,
# travels to the GPU box with gpurun).  Test/bench infrastructure only: the
# product never imports it.  The reference tree is read-only, so pip builds from
# a scratch copy under /tmp; nothing from the reference is copied into the repo
# history.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
src="${1:-/root/reference/pkg}"
if [ ! -d "$src" ]; then
  echo "reference tree $src absent; keeping prebuilt oracle/_ref" >&2
  exit 0
fi
tmp="$(mktemp -d /tmp/color_ref_build.XXXXXX)"
trap 'rm -rf "$tmp"' EXIT
cp -r "$src" "$tmp/pkg"
rm -rf "$here/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --target "$here/_ref" "$tmp/pkg"
python - "$here/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
from color_rl import kernels
assert "cy" in kernels.available_backends(), "Cython backend did not build"
print("oracle/_ref: color_rl built, backends =", kernels.available_backends())
PY
