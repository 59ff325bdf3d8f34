#!/usr/bin/env bash
# Install the unmodified reference package (fodeabm) into baseline/_ref for the
# base contract's reference arm and tests/test_gpu_plugin.py.
# Offline: --no-index from the wheelhouse, --no-deps (NumPy is in the image).
# The build writes into its source tree, so it installs from a copy under /tmp.
# Idempotent: does nothing when baseline/_ref/fodeabm already exists.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
DEST="$ROOT/baseline/_ref"
if [ -d "$DEST/fodeabm" ]; then
  exit 0
fi
if [ ! -f "$SRC/pyproject.toml" ]; then
  echo "install_reference: no reference at $SRC (skipped)" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/fodeabm_src.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC/." "$TMP/"
python -m pip install -q --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$DEST" "$TMP"
