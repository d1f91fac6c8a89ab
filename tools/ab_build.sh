# Build build/head (git HEAD) and build/cur (working tree) variant libraries for tools/ab_head.sh.
set -e
rm -rf build /tmp/ab_head_wt
git worktree add -f /tmp/ab_head_wt HEAD -q
(cd /tmp/ab_head_wt && bash tools/build_variant.sh head > /dev/null)
mkdir -p build/head && cp /tmp/ab_head_wt/build/head/libgtree_b200.so build/head/
git worktree remove --force /tmp/ab_head_wt
bash tools/build_variant.sh cur > /dev/null
