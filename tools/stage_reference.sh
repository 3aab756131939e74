#!/bin/sh
# Offline install of the UNMODIFIED reference (btasel) into baseline/_ref --
# git-ignored, not gpurun-ignored, so it travels to the GPU box -- plus the
# reference's own test files (baseline/_ref/tests), which
# tests/test_gpu_reference_suite.py runs against this package through the
# tests/refshim `btasel` alias.  Run in the build container (needs
# /root/reference); the GPU box only uses the staged copy.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
if [ ! -d "$ROOT/baseline/_ref/btasel" ]; then
  TMP=$(mktemp -d)
  cp -r "$SRC" "$TMP/pkg"   # the build writes into the source tree; /root/reference is read-only
  python -m pip install --no-index --no-build-isolation --no-deps --target "$ROOT/baseline/_ref" "$TMP/pkg"
  rm -rf "$TMP"
fi
rm -rf "$ROOT/baseline/_ref/tests"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/tests"
find "$ROOT/baseline/_ref/tests" -name __pycache__ -prune -exec rm -rf {} +
echo "staged: $(ls "$ROOT/baseline/_ref")"
