#!/usr/bin/env bash
# Install the UNMODIFIED reference package (hiera2a 0.1.0, numpy-only) into
# oracle/_ref so bench.py's CPU legs can time the reference's own
# optimal_dimension / select_swap on the GPU box (where /root/reference does
# not exist).  oracle/_ref is git-ignored (no reference source enters the
# history) but not gpurun-ignored, so it travels with the snapshot.
# Test/bench infrastructure only: the product never imports it.
set -euo pipefail
REF=${1:-/root/reference/pkg}
HERE=$(cd "$(dirname "$0")" && pwd)
[ -d "$REF" ] || { echo "no reference at $REF; keeping the existing oracle/_ref" >&2; exit 0; }
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF" "$TMP/src"             # the build writes into its source tree; REF is read-only
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --target "$HERE/_ref" "$TMP/src"
python -c "import sys; sys.path.insert(0, '$HERE/_ref'); import hiera2a; print('oracle/_ref: hiera2a', hiera2a.__file__)"
