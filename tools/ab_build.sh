#!/bin/bash
# dev helper: build tools/ab/lib_base.so from git HEAD (a worktree under /tmp) and
# tools/ab/lib_new.so from the working tree, for tools/ab.sh on the GPU box.
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/ab
rm -rf /tmp/ab_base && git worktree prune && git worktree add -f /tmp/ab_base HEAD >/dev/null 2>&1
(cd /tmp/ab_base/paper_1910_02270_b200 && python build.py >/dev/null)
cp /tmp/ab_base/paper_1910_02270_b200/_build/libltfb_gpu.so tools/ab/lib_base.so
git worktree remove --force /tmp/ab_base
(cd paper_1910_02270_b200 && python build.py >/dev/null)
cp paper_1910_02270_b200/_build/libltfb_gpu.so tools/ab/lib_new.so
echo built base and new
