#!/usr/bin/env bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored,
# not gpurun-ignored: it travels to the GPU box with the snapshot) and stage
# its own test suite beside it (baseline/_ref/pkg_tests), so the GPU tests
# can drive the reference's dispatch, tests, selftest and bench harness with
# the b200 kernel registered (tests/test_gpu_ref_hw.py) and bench.py's
# reference arm can run the real numba kernel.  Run here (the container that
# has /root/reference); nothing on the GPU box reads /root/reference.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF="${POSPOPCNT_REF_SRC:-/root/reference/pkg}"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF" "$TMP/pkg"   # the build writes into its source tree; /root/reference is read-only
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" >/dev/null
cp -r "$REF/tests" "$ROOT/baseline/_ref/pkg_tests"
find "$ROOT/baseline/_ref" -name __pycache__ -prune -exec rm -rf {} +
echo "staged: $(ls "$ROOT/baseline/_ref")"
