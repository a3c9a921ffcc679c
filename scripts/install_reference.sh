#!/usr/bin/env bash
# Install the UNMODIFIED reference package (attncast, pure Python) into the git-ignored baseline/_ref,
# plus its own test files, from /root/reference (build container only; baseline/_ref then travels to
# the GPU box with the gpurun snapshot).  Used by:
#   - bench.py --impl reference / cpu_baseline (the reference as shipped: attncast.selector.step)
#   - tests/test_gpu_reference_suite.py (the reference's own test suite against this package)
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no /root/reference: keeping the existing baseline/_ref" >&2; exit 0; }
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/refpkg"          # the reference tree is read-only; the build writes egg-info
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/refpkg" >/dev/null
mkdir -p "$ROOT/baseline/_ref/tests"
cp "$SRC"/tests/*.py "$ROOT/baseline/_ref/tests/"
rm -rf "$TMP"
echo "installed reference into $ROOT/baseline/_ref"
