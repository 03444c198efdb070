#!/bin/bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored, travels to the GPU box
# with the gpurun snapshot; /root/reference itself does not exist there), plus a copy of its test
# suite for tests/ref_compat (the reference's own numerical-path tests run against the drop-in).
# Build container only.  Never committed.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
cp -r /root/reference/pkg "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" > "$TMP/pip.log" 2>&1 || {
  echo "pip install failed (see $TMP/pip.log); copying the pure-Python package instead"
  mkdir -p "$ROOT/baseline/_ref" && cp -r "$TMP/pkg/src/bsesolve" "$ROOT/baseline/_ref/"
}
mkdir -p "$ROOT/baseline/_ref/ref_tests"
cp "$TMP"/pkg/tests/*.py "$ROOT/baseline/_ref/ref_tests/"
rm -rf "$TMP"
echo "reference installed: $(ls "$ROOT/baseline/_ref")"
