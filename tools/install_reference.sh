#!/usr/bin/env bash
# Install the UNMODIFIED reference package (slosim, /root/reference/pkg) into the
# git-ignored baseline/_ref, from a /tmp copy (the reference tree is read-only
# and setuptools writes build files next to the sources).  Offline: no index,
# no build isolation, no dependency resolution (numpy / scipy are in the image).
# baseline/_ref is NOT gpurun-ignored, so it travels to the GPU box, where the
# Level-1 drop-in test and the reference arm of bench.py import it.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
[ -f "$SRC/pyproject.toml" ] || { echo "no reference package at $SRC" >&2; exit 1; }
TMP="$(mktemp -d /tmp/slosim_src.XXXXXX)"
cp -r "$SRC/." "$TMP/"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$ROOT/baseline/_ref" "$TMP"
rm -rf "$TMP"
python - "$ROOT/baseline/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import slosim, slosim.simengine, slosim.report  # noqa: F401  (scipy via slosim.predictor)
print("installed", slosim.__file__)
PY
