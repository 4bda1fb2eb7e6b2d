#!/usr/bin/env bash
# ORACLE - TEST INFRASTRUCTURE ONLY.
# Builds the unmodified reference package (chebjac, with its optional Cython
# kernel _kernels_cy.pyx compiled -O3 by its own setup.py) from the sources
# under /root/reference into oracle/_ref/.  The build writes into its source
# tree, so it runs from a scratch copy under /tmp; nothing from the reference
# is committed (oracle/_ref/ is git-ignored but travels to the GPU box).
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
SRC="${REFERENCE_ROOT:-/root/reference}/pkg"
if [ ! -d "$SRC" ]; then
  echo "reference sources not found at $SRC; keeping existing oracle/_ref" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/chebjac_ref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$HERE/_ref" "$TMP/pkg"
python - <<EOF
import sys; sys.path.insert(0, "$HERE/_ref")
import chebjac
assert "cython" in chebjac.available_backends(), "Cython kernel did not build"
print("oracle/_ref: chebjac", chebjac.__version__, "backends", sorted(chebjac.available_backends()))
EOF
