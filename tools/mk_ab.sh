#!/bin/bash
# Build the committed HEAD into _ab/old (git-ignored, travels with gpurun) for same-box A/B runs (tools/ab.sh).
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/abold _ab/old
git worktree prune
git worktree add -f /tmp/abold HEAD -q
(cd /tmp/abold && python -m paper_1508_07953_b200.build >/dev/null && make -s -C oracle >/dev/null 2>&1 || true)
mkdir -p _ab/old
(cd /tmp/abold && tar cf - --exclude=.git .) | (cd _ab/old && tar xf -)
git worktree remove --force /tmp/abold
echo "built $(git rev-parse --short HEAD) into _ab/old"
