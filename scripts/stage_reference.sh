#!/usr/bin/env bash
# Stage the UNMODIFIED reference package (swdft, /root/reference/pkg) into the
# git-ignored baseline/_ref/ with the offline wheelhouse, as the task's reference-arm
# recipe says.  The reference's build writes into its source tree, so it is installed
# from a copy under /tmp.  baseline/_ref travels to the GPU box with the gpurun snapshot
# (git-ignored, not gpurun-ignored); it is used by
#   integration/swdft_b200.py's test (the reference's own tree_swdft_2d backed by
#   libswdft2d.so) and bench.py's numpy-reference CPU timing.
# Usage: scripts/stage_reference.sh [reference_root]   (default /root/reference)
set -euo pipefail
REF=${1:-/root/reference}
HERE=$(cd "$(dirname "$0")/.." && pwd)
DEST="$HERE/baseline/_ref"
if [ ! -d "$REF/pkg/src/swdft" ]; then
  echo "stage_reference: $REF/pkg/src/swdft not found" >&2
  exit 1
fi
TMP=$(mktemp -d /tmp/swdft_ref.XXXXXX)
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF/pkg" "$TMP/pkg"
rm -rf "$DEST"
mkdir -p "$DEST"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$DEST" "$TMP/pkg"
test -f "$DEST/swdft/tree2d.py"
echo "staged swdft into $DEST"
