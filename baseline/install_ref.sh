#!/usr/bin/env bash
# Install the UNMODIFIED reference (walkvec, /root/reference/pkg) into baseline/_ref.
# baseline/_ref is git-ignored but not gpurun-ignored, so it travels to the GPU box,
# where /root/reference does not exist.  Used by bench.py --impl reference (the
# reference's own functions on the host cores) and tests/test_gpu_conformance.py
# (the reference's own test-suite run against the B200 backend through install()).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
src="${1:-/root/reference/pkg}"
tmp="$(mktemp -d)"
trap 'rm -rf "$tmp"' EXIT
cp -r "$src" "$tmp/pkg"  # /root/reference is read-only; setuptools writes build/ and egg-info
rm -rf "$here/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$here/_ref" "$tmp/pkg"
# the reference's own test-suite (+ its oracles, fixtures and data files), unmodified
cp -r "$src/tests" "$here/_ref/walkvec_tests"
echo "installed: $(ls "$here/_ref")"
