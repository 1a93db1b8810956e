#!/bin/bash
# Builds the committed HEAD (or the given revision) as paper_2603_25120_b200/libdflop_base.so for
# A/B timing against the working tree (tools/ab_env.sh ... "DFLOP_LIB=paper_2603_25120_b200/libdflop_base.so").
set -e
REV=${1:-HEAD}
R=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/dflop_base && git -C "$R" worktree add -f /tmp/dflop_base "$REV" -q
(cd /tmp/dflop_base && python -c "from paper_2603_25120_b200 import _build; _build.build(force=True)")
cp /tmp/dflop_base/paper_2603_25120_b200/libdflop.so "$R/paper_2603_25120_b200/libdflop_base.so"
git -C "$R" worktree remove --force /tmp/dflop_base
