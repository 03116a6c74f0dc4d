#!/bin/bash
# Install the unmodified reference package (pure Python) into baseline/_ref
# (git-ignored; it travels to the GPU box with the repo snapshot) so that
# tests/test_gpu_integration.py can run the reference's own CLI rebound onto
# libtidq.  Build container only: /root/reference is read-only, so the build
# runs from a copy under /tmp.
set -eu
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP/pkg"
rm -rf "$TMP"
