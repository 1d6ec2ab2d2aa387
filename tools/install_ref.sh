#!/bin/bash
# Install the UNMODIFIED reference (signadd 0.1.0) into baseline/_ref (git-ignored,
# travels to the GPU box with the gpurun snapshot), plus an unmodified copy of its
# own test suite in baseline/_ref/ref_tests for the drop-in conformance run
# (tests/test_ref_conformance.py).  /root/reference is read-only: build from a
# /tmp copy.  Nothing here is committed.
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=${1:-/root/reference/pkg}
[ -d "$SRC" ] || { echo "install_ref: $SRC absent; skipped"; exit 0; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/ref_tests"
# the reference's own recorded CPU outcomes (the conformance run must reproduce them)
cp "$SRC/test_output.txt" "$ROOT/baseline/_ref/ref_tests/reference_test_output.txt"
rm -rf "$TMP"
echo "install_ref: signadd installed into baseline/_ref (+ ref_tests)"
