#!/bin/bash
# Build libgdp2d.so at a git revision into abtmp/libgdp2d_<name>.so (A/B runs).
#   bash tools/build_variant.sh <rev> <name>
set -e
REV=$1; NAME=$2
R=$(cd "$(dirname "$0")/.." && pwd)
WT=/tmp/gdp2d_wt_$NAME
rm -rf "$WT"; git -C "$R" worktree prune
git -C "$R" worktree add -f --detach "$WT" "$REV" >/dev/null
(cd "$WT" && python -c "from paper_2007_00324_b200 import build; build.build_cuda(force=True)" >/dev/null)
mkdir -p "$R/abtmp"; cp "$WT/paper_2007_00324_b200/lib/libgdp2d.so" "$R/abtmp/libgdp2d_$NAME.so"
git -C "$R" worktree remove --force "$WT"
echo "$R/abtmp/libgdp2d_$NAME.so"
