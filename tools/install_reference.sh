#!/bin/bash
# Install the UNMODIFIED reference package (doublep 0.1.0, Cython backend) into
# baseline/_ref -- the reference arm of bench.py and the integration tests.
# git-ignored, not gpurun-ignored: it travels to the GPU box with the snapshot.
# The build writes into its source tree, so it runs from a copy under /tmp.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
# the reference's own test suite, run against the B200 operators by
# tests/test_gpu_integration.py (through tests/b200_ref_plugin.py)
cp -r "$SRC/tests" "$ROOT/baseline/_ref/tests"
rm -rf "$TMP"
PYTHONPATH="$ROOT/baseline/_ref" python -c "import doublep; print('doublep', doublep.__file__, 'backend', doublep.BACKEND)"
