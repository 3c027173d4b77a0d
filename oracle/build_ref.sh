#!/bin/sh
# Installs the UNMODIFIED reference package (pure Python: /root/reference/pkg, package
# `gausstrack`) into oracle/_ref/ -- test infrastructure only, git-ignored, not gpurun-ignored, so
# it travels to the GPU box where /root/reference does not exist.  Used by the drop-in test
# (tests/test_gpu_dropin.py): the reference's own compensate_frame with and without
# paper_2604_02586_b200.patch.install().  The reference tree is read-only, so pip builds from a
# copy under /tmp.  No reference source is committed to this repository.
set -e
REF=${REF:-/root/reference/pkg}
HERE=$(cd "$(dirname "$0")" && pwd)
[ -d "$REF" ] || { echo "build_ref: $REF absent, keeping oracle/_ref as is"; exit 0; }
TMP=$(mktemp -d)
cp -r "$REF" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install -q --no-index --no-deps --no-build-isolation --target "$HERE/_ref" "$TMP/pkg"
rm -rf "$TMP"
echo "build_ref: gausstrack installed into $HERE/_ref"
