#!/bin/bash
# Build the committed HEAD's library into build/var_head/ (a worktree under
# /tmp), so tools/ab_bench.sh can A/B an uncommitted tree against it:
#   tools/build_head.sh && tools/build_variant.sh mine && SKIPBASE=1 ... ab_bench.sh head mine
set -eu
root=$(git rev-parse --show-toplevel)
wt=$(mktemp -d /tmp/headwt.XXXX)
git -C "$root" worktree add -q --detach "$wt" HEAD
(cd "$wt" && bash tools/build_variant.sh head >/dev/null)
mkdir -p "$root/build/var_head"
cp "$wt/build/var_head/libwarplm_b200.so" "$root/build/var_head/"
git -C "$root" worktree remove --force "$wt"
echo "built build/var_head/libwarplm_b200.so"
