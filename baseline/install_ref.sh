#!/bin/bash
# Install the UNMODIFIED reference package (arxiv/paper_2508_02613, `jfft`)
# into baseline/_ref (git-ignored; it travels to the GPU box with the
# snapshot).  The offline wheelhouse has no numpy wheel for dependency
# resolution, so the install runs with --no-deps (numpy is in the image).
# The reference's own test suite is copied next to it so that it can be run
# through paper_2508_02613_b200.plugin on the GPU box
# (tests/run_reference_suite.py), where /root/reference does not exist.
set -euo pipefail
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=${1:-/root/reference}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/ref"
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$HERE/_ref" "$TMP/ref/pkg"
cp -r "$TMP/ref/pkg/tests" "$HERE/_ref/tests"
rm -rf "$TMP"
echo "installed into $HERE/_ref"
