#!/bin/bash
# Build the committed HEAD's library into ab/libscfa_head.so (A/B baseline for scripts/ab.sh).
set -e
rm -rf /tmp/headwt
git -C "$(dirname "$0")/.." worktree add -q /tmp/headwt HEAD
(cd /tmp/headwt && python -c "from paper_2306_01160_b200 import build; build.build(force=True)" > /dev/null)
mkdir -p "$(dirname "$0")/../ab"
cp /tmp/headwt/paper_2306_01160_b200/lib/libscfa_b200.so "$(dirname "$0")/../ab/libscfa_head.so"
git -C "$(dirname "$0")/.." worktree remove --force /tmp/headwt
