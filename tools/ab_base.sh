#!/bin/bash
# A/B helper: check out COMMIT (default HEAD) as a worktree in .ab_base/ (git-ignored, shipped
# to the GPU box by gpurun) and build its library there, so one gpurun call can time both trees
# on the same box:  (cd .ab_base && python bench.py ...)  vs  python bench.py ...
set -e
cd "$(dirname "$0")/.."
rev=${1:-HEAD}
git worktree remove --force .ab_base 2>/dev/null || rm -rf .ab_base
git worktree add --detach .ab_base "$rev" >/dev/null
(cd .ab_base && python -c "import __graft_entry__ as g; g.build()" > /dev/null)
ls -la .ab_base/paper_2602_08387_b200/libb2s.so
