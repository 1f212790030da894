#!/usr/bin/env bash
# Install the UNMODIFIED reference (conegrad 0.1.0, /root/reference/pkg) into
# baseline/_ref with its compiled Cython backend (_kernels/_csc).  Offline:
# the wheelhouse provides setuptools/Cython/numpy; the build writes into the
# source tree, so it runs from a scratch copy (/root/reference is read-only).
# baseline/_ref is git-ignored but travels to the GPU box with gpurun.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$HERE/_ref" "$TMP/pkg" >/dev/null
# the reference's own test suite travels with the install (tests/test_gpu_reference_suite.py
# runs it against the GPU path through integration/conegrad_plugin.py)
cp -r "$SRC/tests" "$HERE/_ref/tests"
PYTHONPATH="$HERE/_ref" python -c "import conegrad._kernels as k; print('conegrad', k.available_backends() if hasattr(k, 'available_backends') else k._BACKENDS.keys())"
